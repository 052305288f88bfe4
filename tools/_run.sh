timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -1 gpurun_out/ref.json | cut -c1-300
