mkdir -p gpurun_out
for cfg in 2 4 5; do
  timeout 600 python -u bench.py --no-cpu --config $cfg --e2e-steps 1 --steps 5 > gpurun_out/g32_c$cfg.log 2>&1
  echo "cfg$cfg: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g32_c$cfg.log | head -1) $(grep -o '"value": [0-9.e+]*' gpurun_out/g32_c$cfg.log | head -1) $(grep -o '"stages_ms": {[^}]*}' gpurun_out/g32_c$cfg.log)"
  tail -c 300 gpurun_out/g32_c$cfg.log | grep -i "error" | head -2
done
