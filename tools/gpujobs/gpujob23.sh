# A/B of library variants (variants/libdc_v*.so swapped in): owner kernel time (mode 0, 3 runs) + mode 9 split
mkdir -p gpurun_out
cp paper_2411_02797_b200/libdc.so /tmp/libdc_cur.so
for v in 0 1 2 0; do
  cp variants/libdc_v$v.so paper_2411_02797_b200/libdc.so
  timeout 300 python -u tools/own_modes.py 0 0 0 > gpurun_out/g23_v$v.log 2>&1
  echo "v$v: $(grep '"mode"' gpurun_out/g23_v$v.log | tr '\n' ' ')"
  grep "own_split\|own_out\|own_producer" gpurun_out/g23_v$v.log | head -3
done
cp /tmp/libdc_cur.so paper_2411_02797_b200/libdc.so
