# round-1 (g) profiles: bench line, launch list (config 3), config 4 launch list with dram bytes, --set full of the top kernels
# one --set full capture of the top kernels of config 3
mkdir -p gpurun_out
timeout 300 python -u bench.py --steps 20 > gpurun_out/bench_final.log 2>&1; tail -c 3000 gpurun_out/bench_final.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01g_launches.csv python -u bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/r01g_launches.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01g_cfg4_launches.csv python -u bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/r01g_cfg4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pc_owner|k_br_count|k_small_rank|k_intern_rank_small|k_intern_insert|k_path_hash|k_path_group" -s 30 -c 6 -o gpurun_out/r01g_full python -u bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/r01g_full.log 2>&1
ls -la gpurun_out/ | grep r01g
