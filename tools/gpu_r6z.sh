mkdir -p gpurun_out
echo "more division removal" > gpurun_out/r6z_ab.log
timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r6z_ab.log 2>&1
timeout 300 python tools/sinr_real.py C3 64 2 3 >> gpurun_out/r6z_ab.log 2>&1
timeout 300 python tools/sinr_real.py C5 64 2 3 >> gpurun_out/r6z_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r6z_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r6z_pytest.log
