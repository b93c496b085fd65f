mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cfg4_launches.csv python -u bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/cfg4_launches.log 2>&1
tail -c 300 gpurun_out/cfg4_launches.log
