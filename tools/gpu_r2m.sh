mkdir -p gpurun_out
for ws in 0 1; do
GWT_RGRAM_WS=$ws GWT_SINR_DEV_LANES=1 timeout 300 python tools/sinr_time.py C4 2 > gpurun_out/m_time_C4_ws$ws.log 2>&1
GWT_RGRAM_WS=$ws timeout 300 python tools/sinr_time.py C4 2 > gpurun_out/m_time2_C4_ws$ws.log 2>&1
done
GWT_RGRAM_WS=1 timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -q -x -k "sinr" > gpurun_out/m_pytest.log 2>&1
