timeout 120 python tools/e2e_probe.py
