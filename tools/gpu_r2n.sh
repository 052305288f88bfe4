mkdir -p gpurun_out
GWT_SINR_DEV_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n_launch.csv python tools/sinr_once.py C4 128 > gpurun_out/n_ncu1.log 2>&1
GWT_SINR_DEV_LANES=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgram|k_sinr_users|k_esplit" -c 3 -o gpurun_out/n_rg python tools/sinr_once.py C4 64 > gpurun_out/n_ncu2.log 2>&1
