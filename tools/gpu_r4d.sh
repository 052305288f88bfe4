mkdir -p gpurun_out
GWT_LIB_PATH=paper_2401_09792_b200/_build/v2/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 32 2 3 > gpurun_out/r4d_v2.log 2>&1
