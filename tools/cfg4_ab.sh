#!/bin/bash
# Measurement only: config-4 bench step per variant (main = in-tree libdc.so, rows = main with
# DC_PG_ROWS=1, other names = variants/libdc_<name>.so). Usage: bash tools/cfg4_ab.sh TAG v1 v2 ...
T=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  unset DC_PG_ROWS DC_SO_OVERRIDE
  if [ $v = rows ]; then export DC_PG_ROWS=1; elif [ $v != main ]; then export DC_SO_OVERRIDE=$PWD/variants/libdc_$v.so; fi
  timeout 600 python -u bench.py --config 4 --steps 5 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/$T.cfg4_$v.log 2>&1
  tail -c 1500 gpurun_out/$T.cfg4_$v.log | python3 -c "import sys,json; l=[x for x in sys.stdin.read().splitlines() if x.startswith('{')][-1]; d=json.loads(l); print('$v', d['ms_per_step'], {k:v for k,v in d['stages_ms'].items() if k.startswith('k:') or k in ('build','attribute','rollup')})"
done
