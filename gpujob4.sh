timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_modes.csv python -u tools/own_modes.py 0 > gpurun_out/ncu_modes.log 2>&1
tail -3 gpurun_out/ncu_modes.log
