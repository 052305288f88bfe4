mkdir -p gpurun_out
GWT_LIB_PATH=paper_2401_09792_b200/_build/tim/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 32 1 1 2>&1 | sort | uniq -c | sort -rn | head -8 > gpurun_out/r6c_tim.log
echo noepi >> gpurun_out/r6c_tim.log
GWT_LIB_PATH=paper_2401_09792_b200/_build/timpe/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 32 1 1 2>&1 | sort | uniq -c | sort -rn | head -8 >> gpurun_out/r6c_tim.log
