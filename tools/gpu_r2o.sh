mkdir -p gpurun_out
for sp in 0 1; do
GWT_RGRAM_SPLIT=$sp GWT_SINR_DEV_LANES=1 timeout 300 python tools/sinr_time.py C4 2 > gpurun_out/o_time_C4_sp$sp.log 2>&1
GWT_RGRAM_SPLIT=$sp timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -q -x -k "sinr" > gpurun_out/o_pytest_sp$sp.log 2>&1
done
