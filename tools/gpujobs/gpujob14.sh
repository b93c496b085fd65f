mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_push_smem" -s 2 -c 1 -o gpurun_out/push_full python -u bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/push_full.log 2>&1
DC_TEST_ROLLUP_LEVELS=1 timeout 300 python -u bench.py --no-cpu --e2e-steps 1 --steps 30 > gpurun_out/g14_lv.log 2>&1
echo "cfg3 levels: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g14_lv.log | head -1) $(grep -o '"rollup": [0-9.]*' gpurun_out/g14_lv.log)"
ls -la gpurun_out/push_full.ncu-rep
