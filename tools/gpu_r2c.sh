mkdir -p gpurun_out
timeout 600 python tools/diag_tucker.py C4 2 5 > gpurun_out/c_diag.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -k "tucker or solve or trace or nmse or factor or shared or individual" > gpurun_out/c_pytest.log 2>&1
timeout 600 python tools/tucker_time.py C4 64 > gpurun_out/c_tt.log 2>&1
