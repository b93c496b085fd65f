#!/bin/bash
# Measurement only: own_modes.py (k_pc_owner modes) for the in-tree libdc.so ("main") and each
# variants/libdc_<v>.so given, alternating, same box. Usage: bash tools/ab_run.sh TAG "modes" v1 v2 ...
TAG=$1; MODES=$2; shift 2
mkdir -p gpurun_out
for r in 1 2; do
for v in main "$@"; do
  if [ $v = main ]; then unset DC_SO_OVERRIDE; else export DC_SO_OVERRIDE=$PWD/variants/libdc_$v.so; fi
  echo "== $v" >> gpurun_out/$TAG.ab.log
  python tools/own_modes.py $MODES 2>&1 | grep mode >> gpurun_out/$TAG.ab.log
done
done
cat gpurun_out/$TAG.ab.log
