timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
GWT_LIB_PATH=paper_2401_09792_b200/_build/phase/libgwt_b200.so timeout 300 python tools/eig_phases.py 2>&1 | tail -4
timeout 300 python tools/eig_probe.py 2>&1 | tail -4
timeout 300 python tools/tucker_probe.py 2>&1 | tail -4
