timeout 900 python bench.py > gpurun_out/r01_bench.log 2>&1; tail -1 gpurun_out/r01_bench.log > gpurun_out/r01_bench.json; python tools/show_bench.py gpurun_out/r01_bench.json 2>/dev/null | head -6
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file /tmp/r01_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /tmp/ncu_launch.log 2>&1
python tools/ncu_summary.py launches /tmp/r01_launches.csv > gpurun_out/r01_launches.txt; head -28 gpurun_out/r01_launches.txt
GWT_SINR_DEV_LANES=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_rebuild_link|k_pair_gram_gf|k_small_fused" --launch-count 3 -o /tmp/r01_full_sinr -f python tools/sinr_once.py C2 > /tmp/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_heev_cr|k_heev_wr|k_cgemm_conjU|k_gram|k_mode1" --launch-count 10 -o /tmp/r01_full_tucker -f python tools/tucker_once.py C2 64 1 > /tmp/ncu_full_t.log 2>&1
python tools/ncu_summary.py full /tmp/r01_full_sinr.ncu-rep > gpurun_out/r01_ncu_full_sinr.txt
python tools/ncu_summary.py full /tmp/r01_full_tucker.ncu-rep > gpurun_out/r01_ncu_full_tucker.txt
python tools/ncu_lines.py /tmp/r01_full_sinr.ncu-rep 40 > gpurun_out/r01_stall_lines_sinr.txt
