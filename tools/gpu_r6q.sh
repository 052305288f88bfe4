mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r6q_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r6q_pytest.log
timeout 1500 python bench.py > gpurun_out/r6q_bench.json 2> gpurun_out/r6q_bench.err; echo "rc $?" >> gpurun_out/r6q_bench.err
