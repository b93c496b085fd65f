mkdir -p gpurun_out
timeout 600 python -u bench.py --config 5 --steps 5 --e2e-steps 1 --cpu-launches 20000 > gpurun_out/bench_cfg5.log 2>&1
tail -c 2500 gpurun_out/bench_cfg5.log
