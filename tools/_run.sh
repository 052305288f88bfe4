python -m pytest tests/test_gpu_parity.py tests/test_tc.py -x -q 2>&1 | tail -3
for L in 1 2 4; do echo "lanes $L"; GWT_SOLVE_LANES=$L python tools/tucker_probe.py 2>&1 | tail -4; done
