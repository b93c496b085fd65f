# configs 4/5 parity + bench lines for configs 4 and 2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_configs45.py -x -q > gpurun_out/gpu_tests45.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests45.log
tail -15 gpurun_out/gpu_tests45.log
timeout 900 python -u bench.py --config 4 --steps 5 --no-cpu --e2e-steps 0 > gpurun_out/bench_cfg4.log 2>&1
tail -c 2500 gpurun_out/bench_cfg4.log
timeout 900 python -u bench.py --config 2 --steps 10 --no-cpu > gpurun_out/bench_cfg2.log 2>&1
tail -c 2500 gpurun_out/bench_cfg2.log
