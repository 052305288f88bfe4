mkdir -p gpurun_out
echo "warp-local QL, 20 sweeps" > gpurun_out/r6p_ab.log
timeout 300 python tools/sinr_real.py C4 64 20 3 >> gpurun_out/r6p_ab.log 2>&1
timeout 300 python tools/sinr_real.py C3 64 20 3 >> gpurun_out/r6p_ab.log 2>&1
echo "packed QL, 20 sweeps" >> gpurun_out/r6p_ab.log
GWT_LIB_PATH=paper_2401_09792_b200/_build/qlp/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 64 20 3 >> gpurun_out/r6p_ab.log 2>&1
GWT_LIB_PATH=paper_2401_09792_b200/_build/qlp/libgwt_b200.so timeout 300 python tools/sinr_real.py C3 64 20 3 >> gpurun_out/r6p_ab.log 2>&1
echo "packed QL, 2 sweeps" >> gpurun_out/r6p_ab.log
GWT_LIB_PATH=paper_2401_09792_b200/_build/qlp/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r6p_ab.log 2>&1
