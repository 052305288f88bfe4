timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "FAILED|passed|failed" | head -5
for i in 1 2; do echo "tr64 $(timeout 300 python tools/tucker_probe.py 2>&1 | head -1)"; echo "tr128 $(GWT_GEMM_TR64=0 timeout 300 python tools/tucker_probe.py 2>&1 | head -1)"; done
timeout 300 python tools/tucker_probe.py 2>&1 | tail -3
