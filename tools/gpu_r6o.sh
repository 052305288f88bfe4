mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r6o_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r6o_pytest.log
timeout 1500 python bench.py > gpurun_out/r6o_bench.json 2> gpurun_out/r6o_bench.err; echo "rc $?" >> gpurun_out/r6o_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r6o_ref.json 2> gpurun_out/r6o_ref.err; echo "rc $?" >> gpurun_out/r6o_ref.err
