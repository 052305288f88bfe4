mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r7d_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r7d_pytest.log
timeout 300 python tools/sinr_real.py C4 64 2 3 > gpurun_out/r7d_ab.log 2>&1
timeout 300 python tools/sinr_real.py C5 64 2 3 >> gpurun_out/r7d_ab.log 2>&1
timeout 300 python tools/sinr_time.py C2 20 >> gpurun_out/r7d_ab.log 2>&1
