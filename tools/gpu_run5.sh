set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -m gpu -k "sinr" > gpurun_out/r5_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r5_pytest.log
timeout 600 python tools/diag_c4.py C4 8 > gpurun_out/r5_diag.log 2>&1
for c in C4 C3 C5; do GWT_SINR_DEV_LANES=1 timeout 300 python tools/sinr_time.py $c 4 > gpurun_out/r5_time1_$c.log 2>&1; done
for c in C2 C5; do GWT_SINR_PATH=users GWT_SINR_DEV_LANES=1 timeout 300 python tools/sinr_time.py $c 4 > gpurun_out/r5_timeU_$c.log 2>&1; GWT_SINR_DEV_LANES=1 timeout 300 python tools/sinr_time.py $c 4 > gpurun_out/r5_time1_$c.log 2>&1; done
timeout 300 python tools/sinr_once.py C4 64 > gpurun_out/r5_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sinr_users|k_rebuild_mm" -c 2 -o gpurun_out/r5_c4 python tools/sinr_once.py C4 64 > gpurun_out/r5_ncu.log 2>&1
