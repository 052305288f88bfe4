mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r7k_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r7k_pytest.log
timeout 1500 python bench.py > gpurun_out/r7k_bench.json 2> gpurun_out/r7k_bench.err; echo "rc $?" >> gpurun_out/r7k_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r7k_ref.json 2> gpurun_out/r7k_ref.err; echo "rc $?" >> gpurun_out/r7k_ref.err
timeout 900 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r7k_smoke.log 2>&1
