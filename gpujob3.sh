set -x
timeout 300 python -u tools/own_modes.py 0 > gpurun_out/modes.log 2>&1
cat gpurun_out/modes.log | tail -8
timeout 900 python -u -m pytest tests -m gpu -q -x --timeout 200 --timeout-method thread -p no:cacheprovider --tb=short > gpurun_out/gpu_tests.log 2>&1
tail -15 gpurun_out/gpu_tests.log
timeout 900 python -u bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -c 3000 gpurun_out/bench.log
