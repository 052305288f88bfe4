timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "leading or groupwise or large or shared" 2>&1 | tail -2
GWT_LIB_PATH=paper_2401_09792_b200/_build/phase/libgwt_b200.so timeout 120 python tools/eig_phases.py 2>&1 | tail -4
timeout 120 python tools/eig_probe.py 2>&1 | tail -4
timeout 300 python tools/tucker_probe.py 2>&1 | tail -4
