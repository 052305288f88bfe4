mkdir -p gpurun_out
echo "dfma epi, 2p negate" > gpurun_out/r5h_ab.log
GWT_RGRAM_EPI=dfma timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r5h_ab.log 2>&1
GWT_RGRAM_EPI=dfma timeout 300 python tools/sinr_real.py C5 64 2 3 >> gpurun_out/r5h_ab.log 2>&1
echo "dfma epi, 3p" >> gpurun_out/r5h_ab.log
GWT_RGRAM_BK3=1 GWT_RGRAM_EPI=dfma timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r5h_ab.log 2>&1
GWT_RGRAM_BK3=1 GWT_RGRAM_EPI=dfma timeout 300 python tools/sinr_real.py C5 64 2 3 >> gpurun_out/r5h_ab.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgram" -c 1 -o gpurun_out/r5h_rg python tools/sinr_real.py C4 32 1 1 > gpurun_out/r5h_ncu.log 2>&1
