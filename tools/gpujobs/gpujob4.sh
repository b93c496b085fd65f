mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs45.py -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
DC_BUILD_SPLIT_VERIFY=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs45.py -x -q --timeout 300 > gpurun_out/gpu_tests_split.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_split.log
tail -2 gpurun_out/gpu_tests.log gpurun_out/gpu_tests_split.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cfg4_launches.csv python -u bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/cfg4_launches.log 2>&1
