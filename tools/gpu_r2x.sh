mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tc.py tests/test_gpu_scale.py -m gpu -q -x -k "tc or tucker" > gpurun_out/x_pytest.log 2>&1
timeout 600 python tools/tucker_time.py C4 64 > gpurun_out/x_tt4.log 2>&1
timeout 600 python tools/diag_tucker.py C4 2 5 > gpurun_out/x_diag.log 2>&1
timeout 600 python tools/tucker_time.py C3 64 > gpurun_out/x_tt3.log 2>&1
timeout 600 python tools/tucker_time.py C5 128 > gpurun_out/x_tt5.log 2>&1
GWT_GRAM_TC=0 timeout 600 python tools/tucker_time.py C4 64 > gpurun_out/x_tt4_simt.log 2>&1
