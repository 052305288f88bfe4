for c in C2 C2d C1 C2; do echo "== $c $(GWT_SINR_DEV_LANES=1 timeout 120 python tools/sinr_time.py $c 20 | tail -1)"; done
echo "== C2 2 lanes $(timeout 120 python tools/sinr_time.py C2 50 | tail -1)"
