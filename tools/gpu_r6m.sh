mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sinr_users" -c 1 -o gpurun_out/r6m_users python tools/sinr_real.py C4 32 1 1 > gpurun_out/r6m_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgram" -c 1 -o gpurun_out/r6m_rg python tools/sinr_real.py C4 32 1 1 >> gpurun_out/r6m_ncu.log 2>&1
