mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_merge.py -x -q --timeout 300 > gpurun_out/g19_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g19_tests.log
tail -3 gpurun_out/g19_tests.log; grep -m3 "Error\|assert" gpurun_out/g19_tests.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1200 -k "skewed or high_cardinality or generic_schedule" > gpurun_out/san_memcheck4.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck4.log
tail -2 gpurun_out/san_memcheck4.log; grep -m3 "Invalid" gpurun_out/san_memcheck4.log
timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 50 > gpurun_out/g19_b.log 2>&1
echo "cfg3: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g19_b.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/g19_b.log) $(grep -o '"step_ms_dist": {[^}]*}' gpurun_out/g19_b.log)"
