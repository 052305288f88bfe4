timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "sinr or pipeline or end_to_end or large or device" 2>&1 | tail -2
for v in 0 1; do if [ $v = 1 ]; then export GWT_SMALL_SPLIT=1; fi; GWT_SINR_DEV_LANES=1 timeout 120 python tools/sinr_time.py C2 40 2>&1 | tail -1; done
