timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pc_owner" -s 3 -c 1 -o gpurun_out/prof_owner3 python -u bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/ncu_full3.log 2>&1
ls -la gpurun_out/prof_owner3.ncu-rep
