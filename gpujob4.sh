mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -u tools/own_modes.py 9 0 > gpurun_out/own_modes.log 2>&1
grep -v "^$" gpurun_out/own_modes.log | tail -6
for i in 1 2; do timeout 300 python -u bench.py --steps 20 --no-cpu --e2e-steps 0 > gpurun_out/bench_$i.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*' gpurun_out/bench_$i.log; done
grep -o '"stages_ms": {[^}]*}' gpurun_out/bench_2.log
