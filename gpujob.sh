set -x
timeout 300 python -u -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -u -m pytest tests -m gpu -v --timeout 200 --timeout-method thread -p no:cacheprovider --tb=short > gpurun_out/gpu_tests.log 2>&1
grep -E "PASSED|FAILED|ERROR|Timeout|passed|failed" gpurun_out/gpu_tests.log | tail -40
timeout 600 python -u bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -c 2500 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python -u bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pc_owner|k_own_reduce" -s 6 -c 2 -o gpurun_out/prof_owner2 python -u bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
