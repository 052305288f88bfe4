timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/b$i.json 2>/dev/null; python tools/show_bench.py gpurun_out/b$i.json | head -1; done
for i in 1 2; do GWT_SINR_COPY_STREAMS=0 timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/c$i.json 2>/dev/null; python tools/show_bench.py gpurun_out/c$i.json | head -1; done
