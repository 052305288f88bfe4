python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b_def.log 2>&1; python tools/show_bench.py gpurun_out/b_def.log 2>&1 | head -4
for n in 1 4 16; do GWT_SINR_PIPELINE=$n python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_p$n.log 2>&1; echo "pipeline $n"; python tools/show_bench.py gpurun_out/b_p$n.log 2>&1 | head -1; done
