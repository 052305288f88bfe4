mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -k "eigen or solve or tucker or nmse or Tucker" > gpurun_out/r7j_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r7j_pytest.log
timeout 300 python tools/tucker_time.py C4 64 > gpurun_out/r7j_tucker.log 2>&1
timeout 300 python tools/tucker_time.py C2d >> gpurun_out/r7j_tucker.log 2>&1
timeout 300 python tools/tucker_time.py C2 >> gpurun_out/r7j_tucker.log 2>&1
