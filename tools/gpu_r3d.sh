mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -q -x -k "sweep" > gpurun_out/d3_pytest.log 2>&1
timeout 1800 python bench.py > gpurun_out/d3_bench.json 2> gpurun_out/d3_bench.err
