mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -q -x -k "sinr" > gpurun_out/l_pytest.log 2>&1
for c in C4 C3; do timeout 300 python tools/sinr_time.py $c 3 > gpurun_out/l_time_$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_launch.csv python tools/sinr_once.py C4 32 > gpurun_out/l_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgram" -c 1 -o gpurun_out/l_rg python tools/sinr_once.py C4 32 > gpurun_out/l_ncu.log 2>&1
