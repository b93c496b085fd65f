#!/bin/bash
# End-of-round evidence run (one gpurun call): GPU tests, smoke, the default bench line, the
# other configs' lines, the config-3 launch list, --set full of the dominant kernels of
# configs 3 and 4.   gpurun --timeout 3000 -- 'bash tools/prof_final.sh TAG'
T=${1:-final}
mkdir -p gpurun_out
bash tools/gpujob.sh $T smoke tests bench launches
for a in "--config,4,--steps,5" "--config,2,--steps,20" "--aggregated,--steps,20" "--stress,--steps,5" "--config,4,--records,100000000,--steps,5"; do
  bash tools/gpujob.sh $T "bench:$a,--no-cpu,--e2e-steps,0"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pc_owner|k_ctx_hist|k_ctx_emit|k_roll_cols" -s 20 -c 4 \
  -o gpurun_out/$T.full python -u bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/$T.full.log 2>&1; tail -2 gpurun_out/$T.full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_path_group|k_path_hash|k_attribute" -s 10 -c 3 \
  -o gpurun_out/$T.cfg4full python -u bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/$T.cfg4full.log 2>&1; tail -2 gpurun_out/$T.cfg4full.log
