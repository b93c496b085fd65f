# round-1 (b) profiles: bench variance check, launch list of the bench command, one --set full capture of the top kernels
mkdir -p gpurun_out
for i in 1 2; do timeout 300 python -u bench.py --steps 20 --no-cpu --e2e-steps 0 > gpurun_out/bench_$i.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_$i.log; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b_launches.csv python -u bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/r01b_launches.log 2>&1
tail -c 300 gpurun_out/r01b_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pc_owner|k_br_count|k_br_bits|k_build_small|k_br_emit|k_path_hash|k_path_group" -s 30 -c 7 -o gpurun_out/r01b_full python -u bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/r01b_full.log 2>&1
tail -c 300 gpurun_out/r01b_full.log
ls -la gpurun_out/ | grep r01b
