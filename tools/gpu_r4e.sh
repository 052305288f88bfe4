mkdir -p gpurun_out
V3=paper_2401_09792_b200/_build/v3/libgwt_b200.so
GWT_LIB_PATH=$V3 timeout 300 python tools/sinr_real.py C4 32 2 3 > gpurun_out/r4e_v3.log 2>&1
GWT_LIB_PATH=$V3 timeout 300 python tools/sinr_real.py C3 32 2 3 >> gpurun_out/r4e_v3.log 2>&1
timeout 300 python tools/sinr_real.py C3 32 2 3 >> gpurun_out/r4e_v3.log 2>&1
GWT_LIB_PATH=$V3 timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -x -k "sinr or pipeline or c2 or C2" > gpurun_out/r4e_pytest.log 2>&1
