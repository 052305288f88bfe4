mkdir -p gpurun_out
for d in 64 256; do
GWT_EIG64_MIN_D=$d timeout 600 python tools/diag_tucker.py C4 2 5 > gpurun_out/d_diag_$d.log 2>&1
GWT_EIG64_MIN_D=$d timeout 600 python tools/diag_tucker.py C3 2 8 > gpurun_out/d_diag3_$d.log 2>&1
GWT_EIG64_MIN_D=$d timeout 600 python tools/tucker_time.py C4 64 > gpurun_out/d_tt_$d.log 2>&1
done
timeout 600 python tools/tucker_time.py C4 64 > gpurun_out/d_tt_def.log 2>&1
timeout 600 python tools/diag_tucker.py C3 2 8 > gpurun_out/d_diag3_def.log 2>&1
