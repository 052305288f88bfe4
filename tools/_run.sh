timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 200 python tools/es_probe.py 2>&1 | tail -4
