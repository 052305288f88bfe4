python -m pytest tests/test_tc.py -x -q 2>&1 | tail -2
GWT_LIB_PATH=paper_2401_09792_b200/_build/phase/libgwt_b200.so python tools/eig_phases.py 2>&1 | tail -5
python tools/eig_probe.py 2>&1 | tail -5
GWT_GRAM_TC=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tk_C4.csv python tools/tucker_once.py C4 4 1 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/tk_C4.csv 2>&1 | head -14
