set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -m gpu -k "sinr" > gpurun_out/r4_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4_pytest.log
timeout 600 python tools/diag_c4.py C4 8 > gpurun_out/r4_diag.log 2>&1
for c in C2 C4; do GWT_SINR_DEV_LANES=1 timeout 300 python tools/sinr_time.py $c 5 > gpurun_out/r4_time1_$c.log 2>&1; timeout 300 python tools/sinr_time.py $c 5 > gpurun_out/r4_time_$c.log 2>&1; done
