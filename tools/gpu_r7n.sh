mkdir -p gpurun_out
echo "paired upper serving stores" > gpurun_out/r7n_ab.log
timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r7n_ab.log 2>&1
timeout 300 python tools/sinr_real.py C3 64 2 3 >> gpurun_out/r7n_ab.log 2>&1
timeout 300 python tools/sinr_real.py C5 64 2 3 >> gpurun_out/r7n_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/r7n_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r7n_pytest.log
