mkdir -p gpurun_out
timeout 300 python -u tools/host_overhead.py > gpurun_out/host.log 2>&1; head -60 gpurun_out/host.log
nproc; cat /proc/cpuinfo | grep "model name" | head -1
