mkdir -p gpurun_out
for v in base v1; do
  if [ $v = base ]; then L=paper_2401_09792_b200/_build/libgwt_b200.so; else L=paper_2401_09792_b200/_build/$v/libgwt_b200.so; fi
  GWT_LIB_PATH=$L timeout 300 python tools/sinr_real.py C4 32 2 3 > gpurun_out/r4b_$v.log 2>&1
done
GWT_LIB_PATH=paper_2401_09792_b200/_build/v1/libgwt_b200.so timeout 600 python -m pytest tests/test_gpu_scale.py -m gpu -q -x -k "large_config_sinr" > gpurun_out/r4b_v1_pytest.log 2>&1
