mkdir -p gpurun_out
timeout 1500 python bench.py --extra C2,C3,C5 > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err; echo "rc $?" >> gpurun_out/p_bench.err
