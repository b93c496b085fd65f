# memcheck over the owner schedule, the large-P builders and the merge (bigger kernels)
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_merge.py -x -q --timeout 2000 -k "generic_schedule or high_cardinality or skewed or large_P or permutation or merge_local_config1 or collision" > gpurun_out/san_memcheck2.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck2.log
tail -3 gpurun_out/san_memcheck2.log; grep -m5 "Invalid\|ERROR SUMMARY" gpurun_out/san_memcheck2.log
