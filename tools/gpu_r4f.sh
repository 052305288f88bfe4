mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4f_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r4f_pytest.log
timeout 300 python tools/tucker_once.py C4 16 2 > gpurun_out/r4f_t.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4f_tucker_launches.csv python tools/tucker_once.py C4 16 2 > gpurun_out/r4f_tncu.log 2>&1
timeout 300 python tools/sinr_time.py C2 20 > gpurun_out/r4f_c2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4f_c2_launches.csv python tools/sinr_time.py C2 2 > gpurun_out/r4f_c2ncu.log 2>&1
