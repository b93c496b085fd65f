#!/bin/bash
# Measurement only: bench-level A/B of variant libraries (variants/libdc_<v>.so, built with
# tools/ab_variant.sh) against the in-tree libdc.so, alternating on one box; prints per run the
# step time, k_pc_owner, the context reduce and the partial-entry count (DC_PC_STATS).
#   bash tools/ab_step.sh TAG v1 v2 ...
T=$1; shift
mkdir -p gpurun_out
for r in 1 2; do for v in main "$@"; do
  unset DC_SO_OVERRIDE; if [ $v != main ]; then export DC_SO_OVERRIDE=$PWD/variants/libdc_$v.so; fi
  DC_PC_STATS=1 timeout 300 python -u bench.py --steps 30 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/$T.$v.$r.log 2>&1
  python - "$v" "gpurun_out/$T.$v.$r.log" <<'PY' | tee -a gpurun_out/$T.summary
import json, sys
v, path = sys.argv[1], sys.argv[2]
L = open(path).read().splitlines()
b = [json.loads(l) for l in L if l.startswith('{"metric"')]
st = [json.loads(l)["pc_stats"] for l in L if l.startswith('{"pc_stats"')]
if not b:
    print(v, "FAILED"); sys.exit()
b = b[-1]; s = b["stages_ms"]
print(f"{v:8s} step {b['ms_per_step']:.4f} med {b['step_ms_dist']['median']:.4f} own {s['k:pc_owner']:.4f} "
      f"creduce {s['pc:creduce']:.4f} hist {s.get('k:ctx_hist', 0):.4f} entries {st[-1]['entries'] if st else '?'}")
PY
done; done
