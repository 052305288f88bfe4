mkdir -p gpurun_out
for tc in 0 1; do
GWT_GRAM_TC=$tc timeout 600 python tools/tucker_time.py C4 64 > gpurun_out/u_tt_$tc.log 2>&1
GWT_GRAM_TC=$tc timeout 600 python tools/diag_tucker.py C4 2 5 > gpurun_out/u_diag_$tc.log 2>&1
GWT_GRAM_TC=$tc timeout 600 python tools/tucker_time.py C3 64 > gpurun_out/u_tt3_$tc.log 2>&1
GWT_GRAM_TC=$tc timeout 600 python tools/tucker_time.py C5 128 > gpurun_out/u_tt5_$tc.log 2>&1
done
