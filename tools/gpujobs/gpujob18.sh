mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_configs45.py tests/test_gpu_parity.py tests/test_gpu_merge.py -x -q --timeout 2000 -k "config4_prefix or contended or chunked or with_pc_samples or configs_vs_oracle" > gpurun_out/san_memcheck3.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck3.log
tail -3 gpurun_out/san_memcheck3.log; grep -m5 "Invalid\|ERROR SUMMARY" gpurun_out/san_memcheck3.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1000 -k "f1 or small_build or edge" > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.log
tail -3 gpurun_out/san_racecheck.log; grep -m8 "Race\|hazard\|ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/san_racecheck.log
