GWT_BENCH_DEBUG=1 timeout 400 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -5 gpurun_out/bench.err
