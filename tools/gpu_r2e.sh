mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -q -k "tucker" > gpurun_out/e_pytest.log 2>&1
timeout 600 python tools/tucker_time.py C4 512 > gpurun_out/e_tt.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e_tucker512.csv python tools/tucker_once.py C4 512 1 > gpurun_out/e_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sinr_users -c 1 -o gpurun_out/e_users python tools/sinr_once.py C4 16 > gpurun_out/e_ncu2.log 2>&1
