mkdir -p gpurun_out
for i in 1; do timeout 300 python -u tools/dbg_small.py 2 1000000 2>&1 | grep "DIFF\|error\|duplicate\|N " ; done; echo dbg2-done
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/g11_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g11_tests.log
tail -5 gpurun_out/g11_tests.log
timeout 300 python -u bench.py --no-cpu --config 4 --e2e-steps 1 --steps 5 > gpurun_out/g11_c4.log 2>&1
echo "cfg4: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g11_c4.log | head -1) $(grep -o '"k:path_hash": [0-9.]*' gpurun_out/g11_c4.log) $(grep -o '"build": [0-9.]*' gpurun_out/g11_c4.log)"
timeout 300 python -u bench.py --no-cpu --config 2 --e2e-steps 1 --steps 10 > gpurun_out/g11_c2.log 2>&1
echo "cfg2: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g11_c2.log | head -1) $(grep -o '"build": [0-9.]*' gpurun_out/g11_c2.log)"
