mkdir -p gpurun_out
./tools/micro/dfma_occ > gpurun_out/q_dfma.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -x -k "sinr or pipeline or c2" > gpurun_out/q_pytest.log 2>&1
timeout 600 python tools/sinr_real.py C4 64 2 3 > gpurun_out/q_real_C4.log 2>&1
timeout 600 python tools/sinr_real.py C3 64 2 3 > gpurun_out/q_real_C3.log 2>&1
