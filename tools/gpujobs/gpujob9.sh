mkdir -p gpurun_out
export DC_DEBUG=1
for i in 1 2 3; do timeout 300 python -u tools/dbg_small.py 2 1000000 2>&1 | grep "DIFF\|error\|duplicate" ; done; echo dbg2-done
for i in 1 2; do timeout 300 python -u tools/dbg_small.py 5 2000000 2>&1 | grep "DIFF\|error\|duplicate" ; done; echo dbg5-done
timeout 600 python -m pytest tests/test_gpu_configs45.py -x -q --timeout 300 2>&1 | grep "duplicate\|passed\|failed" | sort | uniq -c | head
