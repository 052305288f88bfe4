mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/z_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/z_ref.json 2> gpurun_out/z_ref.err
