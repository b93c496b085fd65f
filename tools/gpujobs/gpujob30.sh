# outlier check: default bench 3x (50 steps) and 20-step runs 3x, step distributions
mkdir -p gpurun_out
for i in 1 2 3; do
  DC_BENCH_DUMP_STEPS=1 timeout 300 python -u bench.py --no-cpu --e2e-steps 1 > gpurun_out/g30_$i.log 2>&1
  echo "50: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g30_$i.log | head -1) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g30_$i.log)"
  DC_BENCH_DUMP_STEPS=1 timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 20 > gpurun_out/g30s_$i.log 2>&1
  echo "20: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g30s_$i.log | head -1) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g30s_$i.log)"
done
