mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/g28_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g28_tests.log
tail -3 gpurun_out/g28_tests.log; grep -m3 "Error\|assert" gpurun_out/g28_tests.log
for i in 1 2; do
timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 100 > gpurun_out/g28_b.log 2>&1
echo "cfg3: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g28_b.log | head -1) $(grep -o '"k:br_bits": [0-9.]*' gpurun_out/g28_b.log) $(grep -o '"pc:breduce": [0-9.]*' gpurun_out/g28_b.log) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g28_b.log)"
done
