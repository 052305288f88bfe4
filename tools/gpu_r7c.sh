mkdir -p gpurun_out
: > gpurun_out/r7c_ab.log
for v in ql4 ql1; do
echo "variant $v" >> gpurun_out/r7c_ab.log
GWT_LIB_PATH=paper_2401_09792_b200/_build/$v/libgwt_b200.so timeout 200 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r7c_ab.log 2>&1
GWT_QL_PACKED=1 GWT_LIB_PATH=paper_2401_09792_b200/_build/$v/libgwt_b200.so timeout 200 python tools/sinr_real.py C3 64 2 3 >> gpurun_out/r7c_ab.log 2>&1
done
