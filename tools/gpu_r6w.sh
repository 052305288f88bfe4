mkdir -p gpurun_out
echo "A prefetch to L2" > gpurun_out/r6w_ab.log
timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r6w_ab.log 2>&1
timeout 300 python tools/sinr_real.py C3 64 2 3 >> gpurun_out/r6w_ab.log 2>&1
timeout 300 python tools/sinr_real.py C5 64 2 3 >> gpurun_out/r6w_ab.log 2>&1
GWT_LIB_PATH=paper_2401_09792_b200/_build/tim/libgwt_b200.so timeout 300 python tools/sinr_real.py C4 32 1 1 2>&1 | sort | uniq -c | sort -rn | head -3 >> gpurun_out/r6w_ab.log
timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/r6w_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r6w_pytest.log
