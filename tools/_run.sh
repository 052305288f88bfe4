timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for e in 1.0 0.5 0.33; do echo "edge $e"; GWT_SINR_EDGE=$e timeout 300 python tools/e2e_probe.py 2>&1 | tail -5; done
