mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6i_tucker_launches.csv python tools/tucker_once.py C4 64 2 > gpurun_out/r6i_ncu.log 2>&1
