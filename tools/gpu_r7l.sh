mkdir -p gpurun_out
: > gpurun_out/r7l_e2e.log
for n in 4 8 16; do
echo "GWT_SINR_PIPELINE=$n" >> gpurun_out/r7l_e2e.log
GWT_SINR_PIPELINE=$n timeout 600 python tools/e2e_c4.py C4 512 2>&1 | tail -4 >> gpurun_out/r7l_e2e.log
done
