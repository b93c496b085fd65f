mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/g31_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g31_tests.log
tail -3 gpurun_out/g31_tests.log; grep -m3 "Error\|assert" gpurun_out/g31_tests.log
for i in 1 2 3; do
timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 100 > gpurun_out/g31_b.log 2>&1
echo "cfg3: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g31_b.log | head -1) $(grep -o '"build": [0-9.]*' gpurun_out/g31_b.log) $(grep -o '"frac": [0-9.]*' gpurun_out/g31_b.log) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g31_b.log)"
done
