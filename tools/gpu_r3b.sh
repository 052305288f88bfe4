mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tc.py tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -x -k "tc or tucker or trace or solve" > gpurun_out/b3_pytest.log 2>&1
timeout 600 python tools/diag_tucker.py C4 2 5 > gpurun_out/b3_diag.log 2>&1
timeout 600 python tools/tucker_time.py C4 512 > gpurun_out/b3_tt512.log 2>&1
timeout 600 python tools/tucker_time.py C3 256 > gpurun_out/b3_tt3.log 2>&1
timeout 600 python tools/tucker_time.py C5 1024 > gpurun_out/b3_tt5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_tcb" -c 2 -o gpurun_out/b3_gtc python tools/tucker_once.py C4 128 1 > gpurun_out/b3_ncu.log 2>&1
