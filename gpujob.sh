set -x
python -u -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -u -m pytest tests -m gpu -v --timeout 240 -p no:cacheprovider --tb=short > gpurun_out/gpu_tests.log 2>&1
tail -30 gpurun_out/gpu_tests.log
timeout 600 python -u bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -c 2500 gpurun_out/bench.log
