#!/bin/bash
# One parameterised runner for gpurun calls (replaces the round-1 one-off job scripts).
#   gpurun --timeout S -- 'bash tools/gpujob.sh TAG STEP [STEP ...]'
# Steps (outputs under gpurun_out/, prefixed with TAG):
#   build        rebuild every native artefact on the box (same nvcc as here)
#   tests        pytest -m gpu (all GPU parity tests)
#   tests:EXPR   pytest -m gpu -k EXPR
#   smoke        __graft_entry__.smoke()
#   bench        default bench.py line (config 3, 20 steps)
#   bench:ARGS   bench.py with ARGS (commas -> spaces), e.g. bench:--config,4,--steps,5
#   launches     ncu launch list (gpu__time_duration.sum) of 2 default bench steps
#   launches4    ncu launch list + DRAM bytes of one config-4 step
#   full:REGEX   ncu --set full of the kernels matching REGEX in one default bench step
set -u
TAG=$1; shift
mkdir -p gpurun_out
O=gpurun_out/$TAG
for step in "$@"; do
  echo "== $step" >&2
  case $step in
    build) python -c "import __graft_entry__ as g; g.build()" > $O.build.log 2>&1; tail -3 $O.build.log ;;
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > $O.tests.log 2>&1; tail -15 $O.tests.log ;;
    tests:*) timeout 1500 python -m pytest tests -m gpu -x -q -k "${step#tests:}" > $O.tests.log 2>&1; tail -15 $O.tests.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O.smoke.log 2>&1; tail -3 $O.smoke.log ;;
    bench) timeout 400 python -u bench.py --steps 20 --warmup 5 > $O.bench.log 2>&1; tail -c 4000 $O.bench.log ;;
    bench:*) A=${step#bench:}; timeout 900 python -u bench.py ${A//,/ } > $O.bench_${A//[^a-zA-Z0-9]/_}.log 2>&1; tail -c 3000 $O.bench_${A//[^a-zA-Z0-9]/_}.log ;;
    launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O.launches.csv \
                python -u bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu > $O.launches.log 2>&1; tail -2 $O.launches.log ;;
    launches4) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
                --csv --log-file $O.cfg4_launches.csv python -u bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu \
                > $O.cfg4.log 2>&1; tail -2 $O.cfg4.log ;;
    full:*) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${step#full:}" -s 20 -c 8 -o $O.full \
                python -u bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > $O.full.log 2>&1; tail -2 $O.full.log ;;
    *) echo "unknown step $step" ;;
  esac
done
ls -la gpurun_out | grep "$TAG" >&2
