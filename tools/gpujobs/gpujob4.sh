mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "owner or config or f1 or random or generic" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 300 python -u tools/own_modes.py 9 0 > gpurun_out/own_modes.log 2>&1
grep -v "^$" gpurun_out/own_modes.log | tail -6
