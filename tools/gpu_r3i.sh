mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "leading_eigenvectors" > gpurun_out/i3_pytest.log 2>&1
GWT_LIB_PATH=paper_2401_09792_b200/_build/phase/libgwt_b200.so timeout 300 python tools/eig_c4_phases.py 8 > gpurun_out/i3_phases.log 2>&1
timeout 300 python tools/eig_c4_phases.py 32 > gpurun_out/i3_nophase.log 2>&1
timeout 600 python tools/tucker_time.py C4 512 > gpurun_out/i3_tt512.log 2>&1
