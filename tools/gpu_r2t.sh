mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_pytest.log 2>&1
timeout 600 python tools/diag_tucker.py C4 2 5 > gpurun_out/t_diag.log 2>&1
timeout 600 python tools/tucker_time.py C4 64 > gpurun_out/t_tt.log 2>&1
timeout 600 python tools/e2e_c4.py C4 128 > gpurun_out/t_e2e.log 2>&1
