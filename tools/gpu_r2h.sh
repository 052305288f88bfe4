mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgram|k_esplit|k_small_grp" -c 3 -o gpurun_out/h_rg python tools/sinr_once.py C4 4 > gpurun_out/h_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h_launch.csv python tools/sinr_once.py C4 16 > gpurun_out/h_ncu2.log 2>&1
