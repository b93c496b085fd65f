mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l.csv python -u bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/l.log 2>&1
timeout 300 python -u bench.py --steps 20 --no-cpu --e2e-steps 0 > gpurun_out/bench_1.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"step_ms_dist": {[^}]*}' gpurun_out/bench_1.log
