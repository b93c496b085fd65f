mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rules.py -x -q --timeout 300 > gpurun_out/gpu_rules.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_rules.log
tail -8 gpurun_out/gpu_rules.log
