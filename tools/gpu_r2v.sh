mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -x -k "sinr or pipeline or c2" > gpurun_out/v_pytest.log 2>&1
timeout 600 python tools/sinr_real.py C4 64 2 3 > gpurun_out/v_real_C4.log 2>&1
timeout 600 python tools/sinr_real.py C3 64 2 3 > gpurun_out/v_real_C3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_heev_big|k_gram" -c 2 -o gpurun_out/v_big python tools/tucker_once.py C4 16 1 > gpurun_out/v_ncu.log 2>&1
