# small-P build change: full GPU suite, then config-3 bench x2
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/g8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g8_tests.log
tail -4 gpurun_out/g8_tests.log
for i in 1 2; do
  timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 50 > gpurun_out/g8_b$i.log 2>&1
  echo "cfg3: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g8_b$i.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/g8_b$i.log) $(grep -o '"build": [0-9.]*' gpurun_out/g8_b$i.log) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g8_b$i.log)"
done
timeout 300 python -u bench.py --no-cpu --config 2 --e2e-steps 1 --steps 10 > gpurun_out/g8_c2.log 2>&1
echo "cfg2: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g8_c2.log | head -1) $(grep -o '"build": [0-9.]*' gpurun_out/g8_c2.log)"
