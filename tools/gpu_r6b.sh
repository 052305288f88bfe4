mkdir -p gpurun_out
echo "1 pass" > gpurun_out/r6b_ab.log
GWT_LIB_PATH=paper_2401_09792_b200/_build/p1/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r6b_ab.log 2>&1
echo "no epilogue" >> gpurun_out/r6b_ab.log
GWT_LIB_PATH=paper_2401_09792_b200/_build/pe/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r6b_ab.log 2>&1
