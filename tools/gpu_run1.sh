set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r1_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r1_pytest.log
for tc in 0 1 2; do GWT_REBUILD_TC=$tc timeout 300 python tools/sinr_time.py C4 3 > gpurun_out/r1_c4_tc$tc.log 2>&1; done
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/r1_bench.log
