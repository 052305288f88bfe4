timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C2 C1 C5 C3; do echo "== $c $(GWT_SINR_DEV_LANES=1 timeout 120 python tools/sinr_time.py $c 10 | tail -1)"; done
echo "== C2 2 lanes $(timeout 120 python tools/sinr_time.py C2 100 | tail -1)"
