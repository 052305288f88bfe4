set -x
mkdir -p gpurun_out
timeout 600 python tools/diag_c4.py C4 8 > gpurun_out/r3_diag.log 2>&1
timeout 300 python tools/sinr_once.py C4 64 > gpurun_out/r3_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sinr_users|k_rebuild_rb" -c 2 -o gpurun_out/r3_c4 python tools/sinr_once.py C4 64 > gpurun_out/r3_ncu.log 2>&1
