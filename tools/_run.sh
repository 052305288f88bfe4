timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "leading or large" 2>&1 | tail -3
GWT_LIB_PATH=paper_2401_09792_b200/_build/phase/libgwt_b200.so timeout 120 python tools/eig_phases.py 2>&1 | tail -2
timeout 120 python tools/eig_probe.py 2>&1 | tail -1
timeout 300 python tools/tucker_probe.py 2>&1 | tail -4
