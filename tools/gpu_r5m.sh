mkdir -p gpurun_out
GWT_LIB_PATH=paper_2401_09792_b200/_build/tim/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 32 1 1 2>&1 | sort | uniq | tail -4 > gpurun_out/r5m_tim.log
echo late > gpurun_out/r5m_ab.log
timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r5m_ab.log 2>&1
timeout 300 python tools/sinr_real.py C3 64 2 3 >> gpurun_out/r5m_ab.log 2>&1
echo early >> gpurun_out/r5m_ab.log
GWT_RGRAM_LATE=0 timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r5m_ab.log 2>&1
echo late noATS >> gpurun_out/r5m_ab.log
GWT_RGRAM_ATS=0 timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r5m_ab.log 2>&1
