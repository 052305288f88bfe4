python -m pytest tests/test_gpu_parity.py -x -q -k "sinr or pipeline or end_to_end or large" 2>&1 | tail -2
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b_def.log 2>&1; python tools/show_bench.py gpurun_out/b_def.log 2>&1 | head -4
GWT_PG_STAGED=1 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b_st.log 2>&1; python tools/show_bench.py gpurun_out/b_st.log 2>&1 | head -4
