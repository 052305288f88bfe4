mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_tcb" -c 1 -o gpurun_out/y_gtc python tools/tucker_once.py C4 128 1 > gpurun_out/y_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/y_tucker512.csv python tools/tucker_once.py C4 512 1 > /dev/null 2>&1
timeout 600 python tools/tucker_time.py C4 512 > gpurun_out/y_tt512.log 2>&1
