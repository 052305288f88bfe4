mkdir -p gpurun_out
timeout 300 python tools/sinr_real.py C4 64 2 3 > gpurun_out/r5d_ab.log 2>&1
GWT_RGRAM_EPI=dfma timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r5d_ab.log 2>&1
timeout 300 python tools/sinr_real.py C3 64 2 3 >> gpurun_out/r5d_ab.log 2>&1
GWT_RGRAM_EPI=dfma timeout 300 python tools/sinr_real.py C3 64 2 3 >> gpurun_out/r5d_ab.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r5d_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r5d_pytest.log
