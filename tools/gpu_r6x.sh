mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r6x_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r6x_pytest.log
timeout 1500 python bench.py > gpurun_out/r6x_bench.json 2> gpurun_out/r6x_bench.err; echo "rc $?" >> gpurun_out/r6x_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r6x_ref.json 2> gpurun_out/r6x_ref.err; echo "rc $?" >> gpurun_out/r6x_ref.err
timeout 900 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r6x_smoke.log 2>&1
# launch list of the bench command itself (SINR kernels; one timed step)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_rgram|k_esplit|k_bsplit|k_sinr_users" --log-file gpurun_out/r6x_sinr_launches.csv python bench.py --steps 1 --warmup 3 --extra "" --no-cpu-baseline > gpurun_out/r6x_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgram|k_sinr_users|k_esplit" -c 3 -o gpurun_out/r6x_sinr python tools/sinr_real.py C4 32 1 1 > gpurun_out/r6x_ncu2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6x_tucker_launches.csv python tools/tucker_once.py C4 64 1 > gpurun_out/r6x_ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_tcb|k_heev_big|k_cgemm_conjU" -c 6 -o gpurun_out/r6x_tucker python tools/tucker_once.py C4 64 1 > gpurun_out/r6x_ncu4.log 2>&1
