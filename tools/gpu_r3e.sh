mkdir -p gpurun_out
timeout 600 python tools/tucker_once.py C4 128 2 > gpurun_out/e3_once.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e3_tucker_launches.csv python tools/tucker_once.py C4 128 2 > gpurun_out/e3_ncu.log 2>&1
