# A/B of programmatic dependent launch: parity subset, then the config-3 and config-4 bench with/without PDL
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_merge.py tests/test_gpu_rules.py -x -q --timeout 200 > gpurun_out/pdl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdl_tests.log
tail -4 gpurun_out/pdl_tests.log
for i in 1 2; do
  for v in 1 0; do
    DC_NO_PDL=$v timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 50 > gpurun_out/pdl_b$v.log 2>&1
    echo "NO_PDL=$v cfg3: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/pdl_b$v.log) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/pdl_b$v.log)"
  done
done
for v in 1 0; do
  DC_NO_PDL=$v timeout 300 python -u bench.py --no-cpu --config 4 --e2e-steps 1 --steps 5 > gpurun_out/pdl_c4_$v.log 2>&1
  echo "NO_PDL=$v cfg4: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/pdl_c4_$v.log)"
done
tail -c 1500 gpurun_out/pdl_b0.log
