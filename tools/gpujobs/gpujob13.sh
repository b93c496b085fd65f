mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs45.py -x -q --timeout 300 > gpurun_out/g13_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g13_tests.log
tail -3 gpurun_out/g13_tests.log
timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 50 > gpurun_out/g13_b.log 2>&1
echo "cfg3: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g13_b.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/g13_b.log) $(grep -o '"rollup": [0-9.]*' gpurun_out/g13_b.log) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g13_b.log)"
DC_TEST_ROLLUP_PUSH_GLOBAL=1 timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 50 > gpurun_out/g13_bg.log 2>&1
echo "cfg3 global push: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g13_bg.log | head -1) $(grep -o '"rollup": [0-9.]*' gpurun_out/g13_bg.log) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g13_bg.log)"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_push|k_small" --csv python -u bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu 2>/dev/null | grep "k_push\|k_small" | awk -F, '{print $5, $NF}' | head -6
