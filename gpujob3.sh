# new build path: gpu tests + config-4/2/3 bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -25 gpurun_out/gpu_tests.log
timeout 600 python -u bench.py --config 4 --steps 5 --no-cpu --e2e-steps 0 > gpurun_out/bench_cfg4.log 2>&1
tail -c 1800 gpurun_out/bench_cfg4.log
timeout 600 python -u bench.py --config 2 --steps 10 --no-cpu --e2e-steps 0 > gpurun_out/bench_cfg2.log 2>&1
tail -c 1500 gpurun_out/bench_cfg2.log
timeout 600 python -u bench.py --steps 10 --no-cpu --e2e-steps 0 > gpurun_out/bench_cfg3.log 2>&1
tail -c 1500 gpurun_out/bench_cfg3.log
