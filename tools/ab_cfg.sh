#!/bin/bash
# Measurement only: bench-level A/B of variant libraries on one config (alternating, same box).
#   bash tools/ab_cfg.sh TAG "BENCH ARGS" v1 v2 ...   (main = the in-tree libdc.so)
T=$1; A=$2; shift 2
mkdir -p gpurun_out
for r in 1 2; do for v in main "$@"; do
  unset DC_SO_OVERRIDE; if [ $v != main ]; then export DC_SO_OVERRIDE=$PWD/variants/libdc_$v.so; fi
  timeout 600 python -u bench.py $A --no-cpu --e2e-steps 0 > gpurun_out/$T.$v.$r.log 2>&1
  python - "$v" "gpurun_out/$T.$v.$r.log" <<'PY' | tee -a gpurun_out/$T.summary
import json, sys
v, path = sys.argv[1], sys.argv[2]
b = [json.loads(l) for l in open(path) if l.startswith('{"metric"')]
if not b:
    print(v, "FAILED"); sys.exit()
b = b[-1]; s = b["stages_ms"]
print(f"{v:8s} step {b['ms_per_step']:.4f} med {b['step_ms_dist']['median']:.4f} " + " ".join(f"{k} {s[k]:.4f}" for k in ("build", "attribute", "rollup", "pc") if k in s))
PY
done; done
