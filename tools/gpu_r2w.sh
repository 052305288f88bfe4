mkdir -p gpurun_out
for c in 1e-3 1e-4 1e-5; do
GWT_EIG_BIG_CTOL=$c timeout 600 python tools/tucker_time.py C4 64 > gpurun_out/w_tt_$c.log 2>&1
GWT_EIG_BIG_CTOL=$c timeout 600 python tools/diag_tucker.py C4 2 5 > gpurun_out/w_diag_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_heev_big" -c 1 -o gpurun_out/w_big python tools/tucker_once.py C4 16 1 > gpurun_out/w_ncu.log 2>&1
