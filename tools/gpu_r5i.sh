mkdir -p gpurun_out
echo "dfma epi, 2p negate grouped" > gpurun_out/r5i_ab.log
GWT_RGRAM_EPI=dfma timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r5i_ab.log 2>&1
GWT_RGRAM_EPI=dfma timeout 300 python tools/sinr_real.py C5 64 2 3 >> gpurun_out/r5i_ab.log 2>&1
echo "dmma coop, 2p negate grouped" >> gpurun_out/r5i_ab.log
timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r5i_ab.log 2>&1
timeout 300 python tools/sinr_real.py C3 64 2 3 >> gpurun_out/r5i_ab.log 2>&1
