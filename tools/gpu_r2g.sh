mkdir -p gpurun_out
timeout 300 python tools/sinr_once.py C4 4 > gpurun_out/g_once.log 2>&1; echo "rc $?" >> gpurun_out/g_once.log
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -x -k "sinr or pipeline or c2" > gpurun_out/g_pytest.log 2>&1
for c in C4 C2 C5 C3; do timeout 300 python tools/sinr_time.py $c 3 > gpurun_out/g_time_$c.log 2>&1; done
GWT_SINR_PATH=users timeout 300 python tools/sinr_time.py C4 3 > gpurun_out/g_time_C4_users.log 2>&1
