# round-1 profiles: launch list of the bench command + one --set full capture of the top kernels
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python -u bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/r01_launches.log 2>&1
tail -c 400 gpurun_out/r01_launches.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pc_owner|k_br_count|k_br_bits|k_build_small|k_br_emit" -s 20 -c 5 -o gpurun_out/r01_full python -u bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/r01_full.log 2>&1
tail -c 400 gpurun_out/r01_full.log
ls -la gpurun_out/
