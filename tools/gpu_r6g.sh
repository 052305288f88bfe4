mkdir -p gpurun_out
echo "split" > gpurun_out/r6g_ab.log
GWT_RGRAM_SPLIT=1 timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r6g_ab.log 2>&1
