set -x
mkdir -p gpurun_out
bash tools/gpujob.sh r02a bench launches "full:k_pc_owner|k_ctx_hist|k_roll_cols|k_intern_insert|k_small_rank|k_topk_one|k_path_group" launches4
timeout 600 python -u bench.py --config 4 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02a.cfg4.log 2>&1; tail -c 2500 gpurun_out/r02a.cfg4.log
timeout 600 python -u bench.py --config 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/r02a.cfg2.log 2>&1; tail -c 600 gpurun_out/r02a.cfg2.log
timeout 900 python -u bench.py --config 5 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02a.cfg5.log 2>&1; tail -c 600 gpurun_out/r02a.cfg5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_path_group|k_path_hash" -s 6 -c 2 -o gpurun_out/r02a.cfg4full python -u bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/r02a.cfg4full.log 2>&1; tail -2 gpurun_out/r02a.cfg4full.log
