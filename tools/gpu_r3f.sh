mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f3_tucker_launches.csv python tools/tucker_once.py C4 512 1 > gpurun_out/f3_ncu.log 2>&1
