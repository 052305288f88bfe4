timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "FAILED|passed|failed" | head -5
GWT_LIB_PATH=paper_2401_09792_b200/_build/phase/libgwt_b200.so timeout 300 python tools/eig_real_phases.py 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/tucker_probe.py 2>&1 | head -1; done
timeout 300 python tools/tucker_probe.py 2>&1 | tail -3
