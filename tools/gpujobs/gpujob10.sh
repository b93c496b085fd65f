mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python -u tools/dbg_small.py 2 200000 2>&1 | grep "DIFF\|error" ; done; echo dbg-done
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/g10_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g10_tests.log
tail -5 gpurun_out/g10_tests.log
timeout 300 python -u bench.py --no-cpu --config 2 --e2e-steps 1 --steps 10 > gpurun_out/g10_c2.log 2>&1
echo "cfg2: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g10_c2.log | head -1) $(grep -o '"build": [0-9.]*' gpurun_out/g10_c2.log)"
timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 50 > gpurun_out/g10_b.log 2>&1
echo "cfg3: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g10_b.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/g10_b.log) $(grep -o '"build": [0-9.]*' gpurun_out/g10_b.log) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g10_b.log)"
