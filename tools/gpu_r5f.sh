mkdir -p gpurun_out
for ns in 0 400 700 1200 2000; do
echo "stagger $ns" >> gpurun_out/r5f_ab.log
GWT_RGRAM_STAGGER_NS=$ns timeout 300 python tools/sinr_real.py C4 64 2 3 >> gpurun_out/r5f_ab.log 2>&1
done
GWT_RGRAM_STAGGER_NS=700 timeout 300 python tools/sinr_real.py C3 64 2 3 >> gpurun_out/r5f_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/r5f_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r5f_pytest.log
