mkdir -p gpurun_out
timeout 300 python tools/sinr_real.py C4 8 1 1 > gpurun_out/r4c_run.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgram|k_sinr_users" -c 2 -o gpurun_out/r4c_c4 python tools/sinr_real.py C4 8 1 1 > gpurun_out/r4c_ncu.log 2>&1
