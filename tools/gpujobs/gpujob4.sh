mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 300 python -u bench.py --config 2 --steps 10 --no-cpu --e2e-steps 0 > gpurun_out/bench_cfg2.log 2>&1
grep -o '"ms_per_step": [0-9.]*\|"stages_ms": {[^}]*}' gpurun_out/bench_cfg2.log
