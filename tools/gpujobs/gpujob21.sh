mkdir -p gpurun_out
for v in 5 1000 5 1000; do
  DC_BENCH_CLOCK_MS=$v DC_BENCH_DUMP_STEPS=1 timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 200 > gpurun_out/g21_$v.log 2>&1
  echo "clk=$v: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g21_$v.log | head -1) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g21_$v.log)"
  python -c "
import json,re,sys
for l in open('gpurun_out/g21_$v.log'):
    if 'per_step_ms' in l:
        a=json.loads(l)['per_step_ms']; big=[(i,x) for i,x in enumerate(a) if x>1.6]; print('  outliers', big[:12], 'n', len(big))
"
done
