mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sinr_users" -c 1 -o gpurun_out/r7b_users python tools/sinr_real.py C4 32 1 1 > gpurun_out/r7b_ncu.log 2>&1
