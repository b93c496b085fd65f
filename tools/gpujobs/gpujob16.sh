# compute-sanitizer passes over the small GPU tests (memcheck, synccheck), and the suite without PDL
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rules.py -x -q --timeout 900 -k "f1 or random or edge or small_build or dedup or kind_mask or too_deep or collisions or rules or folded or interval or associate or stall" > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
tail -3 gpurun_out/san_memcheck.log; grep -m5 "Invalid\|ERROR SUMMARY\|Error" gpurun_out/san_memcheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "f1 or edge or small_build or skewed" > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_synccheck.log
tail -3 gpurun_out/san_synccheck.log; grep -m5 "ERROR SUMMARY\|Barrier\|error" gpurun_out/san_synccheck.log
DC_NO_PDL=1 timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/nopdl_tests.log 2>&1; echo "nopdl rc=$?" >> gpurun_out/nopdl_tests.log
tail -2 gpurun_out/nopdl_tests.log
