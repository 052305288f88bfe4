timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "leading" 2>&1 | tail -3
