mkdir -p gpurun_out
./tools/micro/dfma_occ > gpurun_out/r5b_dfma.log 2>&1
./tools/micro/dmma > gpurun_out/r5b_dmma.log 2>&1
./tools/micro/f2f > gpurun_out/r5b_f2f.log 2>&1
Q=paper_2401_09792_b200/_build/qlp/libgwt_b200.so
for sw in 2 20; do
timeout 300 python tools/sinr_real.py C4 64 $sw 3 >> gpurun_out/r5b_ab.log 2>&1
GWT_LIB_PATH=$Q timeout 300 python tools/sinr_real.py C4 64 $sw 3 >> gpurun_out/r5b_ab.log 2>&1
done
timeout 300 python tools/sinr_real.py C3 64 20 3 >> gpurun_out/r5b_ab.log 2>&1
GWT_LIB_PATH=$Q timeout 300 python tools/sinr_real.py C3 64 20 3 >> gpurun_out/r5b_ab.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgram|k_sinr_users" -c 2 -o gpurun_out/r5b_c4 python tools/sinr_real.py C4 32 1 1 > gpurun_out/r5b_ncu.log 2>&1
