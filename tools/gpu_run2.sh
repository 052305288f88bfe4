set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2_pytest.log
for c in C2 C4 C3 C5; do timeout 300 python tools/sinr_time.py $c 5 > gpurun_out/r2_time_$c.log 2>&1; done
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/r2_bench.log
