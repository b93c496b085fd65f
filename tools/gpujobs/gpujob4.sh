mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_merge.py -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg2_launches.csv python -u bench.py --config 2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/cfg2_launches.log 2>&1
