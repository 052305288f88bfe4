mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r5a_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r5a_pytest.log
timeout 1200 python bench.py > gpurun_out/r5a_bench.json 2> gpurun_out/r5a_bench.err; echo "rc $?" >> gpurun_out/r5a_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r5a_ref.json 2> gpurun_out/r5a_ref.err; echo "rc $?" >> gpurun_out/r5a_ref.err
