mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s_pytest.log 2>&1
timeout 600 python tools/e2e_c4.py C4 128 > gpurun_out/s_e2e.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_heev_cr" -c 1 -o gpurun_out/s_heev python tools/tucker_once.py C4 4 1 > gpurun_out/s_ncu.log 2>&1
