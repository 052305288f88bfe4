mkdir -p gpurun_out
: > gpurun_out/r6l_ab.log
for v in pc pd pcd pi; do
echo "variant $v" >> gpurun_out/r6l_ab.log
GWT_LIB_PATH=paper_2401_09792_b200/_build/$v/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r6l_ab.log 2>&1
done
