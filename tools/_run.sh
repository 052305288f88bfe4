set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/r01_launches.txt
GWT_SINR_DEV_LANES=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rebuild|k_pair_gram|k_small" -o /tmp/sinr python tools/sinr_once.py C2 > gpurun_out/ncu_sinr.log 2>&1
python tools/ncu_summary.py full /tmp/sinr.ncu-rep > gpurun_out/r01_ncu_full_sinr.txt
python tools/ncu_lines.py /tmp/sinr.ncu-rep 40 > gpurun_out/r01_stall_lines_sinr.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_heev|k_gram|k_cgemm|k_mode1" -c 16 -o /tmp/tucker python tools/tucker_once.py C2 64 1 > gpurun_out/ncu_tucker.log 2>&1
python tools/ncu_summary.py full /tmp/tucker.ncu-rep > gpurun_out/r01_ncu_full_tucker.txt
python tools/ncu_lines.py /tmp/tucker.ncu-rep 40 > gpurun_out/r01_stall_lines_tucker.txt
