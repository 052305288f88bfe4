GWT_LIB_PATH=paper_2401_09792_b200/_build/phase/libgwt_b200.so timeout 300 python tools/eig_real_phases.py 2>&1 | tail -3
