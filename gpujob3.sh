set -x
timeout 300 python -u tools/own_modes.py 0 > gpurun_out/modes.log 2>&1
cat gpurun_out/modes.log | tail -8
timeout 900 python -u -m pytest tests/test_gpu_parity.py tests/test_gpu_merge.py -m gpu -q -x --timeout 200 --timeout-method thread -p no:cacheprovider --tb=short > gpurun_out/gpu_tests.log 2>&1
tail -15 gpurun_out/gpu_tests.log
