mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "leading_eigenvectors" > gpurun_out/g3b_pytest.log 2>&1
GWT_LIB_PATH=paper_2401_09792_b200/_build/phase/libgwt_b200.so timeout 500 python tools/eig_c4_phases.py 8 > gpurun_out/g3b_phases.log 2>&1
timeout 600 python tools/tucker_time.py C4 512 > gpurun_out/g3b_tt512.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_tc.py -m gpu -q -x > gpurun_out/g3b_scale.log 2>&1
