mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
timeout 300 python -u bench.py --config 4 --steps 5 --no-cpu --e2e-steps 0 > gpurun_out/bench_cfg4.log 2>&1
tail -c 1200 gpurun_out/bench_cfg4.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cfg4_launches.csv python -u bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/cfg4_launches.log 2>&1
timeout 300 python -u bench.py --steps 20 > gpurun_out/bench.log 2>&1
tail -c 2500 gpurun_out/bench.log
