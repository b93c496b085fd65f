# variant check: owner parity subset + owner kernel time (mode 0) + mode 9 split
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 200 -k "owner or config3 or pc" > gpurun_out/g7_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g7_tests.log
tail -3 gpurun_out/g7_tests.log
timeout 300 python -u tools/own_modes.py 0 9 0 > gpurun_out/own_modes7.log 2>&1
grep -v "^$" gpurun_out/own_modes7.log | grep -v "^{\"build" | tail -8
