mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c3_pytest.log 2>&1
./paper_2401_09792_b200/_build/test_dropin > gpurun_out/c3_dropin.log 2>&1; echo "rc $?" >> gpurun_out/c3_dropin.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c3_smoke.log 2>&1
timeout 600 python tools/sinr_real.py C4 64 2 3 > gpurun_out/c3_real.log 2>&1
