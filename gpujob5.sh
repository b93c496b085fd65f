timeout 900 python -u bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -c 3000 gpurun_out/bench.log
