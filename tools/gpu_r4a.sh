mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4a_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4a_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r4a_ref.json 2> gpurun_out/r4a_ref.err
