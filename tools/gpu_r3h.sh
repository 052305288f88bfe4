mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "leading_eigenvectors" > gpurun_out/h3_pytest.log 2>&1
for c in 1e-3 1e-4 1e-5; do
GWT_EIG_BIG_CTOL=$c GWT_LIB_PATH=paper_2401_09792_b200/_build/phase/libgwt_b200.so timeout 300 python tools/eig_c4_phases.py 8 > gpurun_out/h3_phases_$c.log 2>&1
done
for c in 1e-3 1e-5; do
GWT_EIG_BIG_CTOL=$c timeout 600 python tools/tucker_time.py C4 512 > gpurun_out/h3_tt512_$c.log 2>&1
done
