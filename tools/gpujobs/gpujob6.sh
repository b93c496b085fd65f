# owner-kernel change check: PC parity subset, per-CTA cycle split, bench config 3 x2
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_merge.py -x -q --timeout 200 -k "owner or pc or config or random or edge or merge" > gpurun_out/g6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g6_tests.log
tail -4 gpurun_out/g6_tests.log
timeout 300 python -u tools/own_modes.py 9 0 > gpurun_out/own_modes.log 2>&1
grep -v "^$" gpurun_out/own_modes.log | tail -6
for i in 1 2; do
  timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 50 > gpurun_out/g6_b$i.log 2>&1
  echo "cfg3: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g6_b$i.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/g6_b$i.log) $(grep -o '"kernel_ms": [0-9.]*' gpurun_out/g6_b$i.log) $(grep -o '"pc:breduce": [0-9.]*' gpurun_out/g6_b$i.log) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g6_b$i.log)"
done
