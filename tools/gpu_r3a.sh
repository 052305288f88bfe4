mkdir -p gpurun_out
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rgram|k_esplit|k_bsplit|k_sinr_users" --csv --log-file gpurun_out/a3_launches.csv python bench.py --steps 1 --warmup 1 --extra "" --no-cpu-baseline > gpurun_out/a3_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rgram|k_sinr_users|k_esplit" -c 3 -o gpurun_out/a3_sinr python tools/sinr_real.py C4 32 1 1 > gpurun_out/a3_ncu.log 2>&1
