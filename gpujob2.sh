timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pc_owner" -s 3 -c 1 -o gpurun_out/prof_owner4 python -u tools/own_modes.py 0 > gpurun_out/ncu_full4.log 2>&1
ls -la gpurun_out/prof_owner4.ncu-rep
