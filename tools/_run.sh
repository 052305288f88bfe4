timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rank_sweep or leading or large" 2>&1 | tail -3
