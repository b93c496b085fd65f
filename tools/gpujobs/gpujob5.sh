mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 200 -k "owner or f1 or config or random or generic or edge" > gpurun_out/gpu_tests_pc.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_pc.log
tail -4 gpurun_out/gpu_tests_pc.log
timeout 300 python -u tools/own_modes.py 9 0 > gpurun_out/own_modes.log 2>&1
grep -v "^$" gpurun_out/own_modes.log | tail -6
