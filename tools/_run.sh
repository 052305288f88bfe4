timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/tucker_probe.py 2>&1 | tail -4
timeout 300 python tools/tucker_probe.py 2>&1 | tail -4 | head -1
