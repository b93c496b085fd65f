mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_merge.py -x -q --timeout 300 -k nccl > gpurun_out/g29_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g29_tests.log
tail -30 gpurun_out/g29_tests.log | grep -v "^$" | tail -15
