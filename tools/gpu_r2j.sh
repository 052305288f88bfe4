mkdir -p gpurun_out
timeout 300 python tools/sinr_once.py C4 4 > gpurun_out/j_once.log 2>&1; echo "rc $?" >> gpurun_out/j_once.log
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -x -k "sinr or pipeline or c2" > gpurun_out/j_pytest.log 2>&1
for c in C4 C3; do timeout 300 python tools/sinr_time.py $c 3 > gpurun_out/j_time_$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_launch.csv python tools/sinr_once.py C4 32 > gpurun_out/j_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgram|k_esplit|k_sinr_users" -c 3 -o gpurun_out/j_rg python tools/sinr_once.py C4 32 > gpurun_out/j_ncu.log 2>&1
