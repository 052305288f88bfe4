mkdir -p gpurun_out
GWT_LIB_PATH=paper_2401_09792_b200/_build/tim/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 32 1 1 > gpurun_out/r5l_tim.log 2>&1
