mkdir -p gpurun_out
timeout 600 python tools/tucker_time.py C4 64 > gpurun_out/r6h_tucker.log 2>&1
timeout 600 python tools/tucker_time.py C3 64 >> gpurun_out/r6h_tucker.log 2>&1
timeout 900 python -m pytest tests/test_tc.py tests/test_gpu_scale.py -m gpu -q -x -k "tc or tucker or Tucker" > gpurun_out/r6h_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r6h_pytest.log
