set -x
mkdir -p gpurun_out
timeout 600 python tools/diag_tucker.py C4 2 5 > gpurun_out/b_diag_def.log 2>&1
GWT_EIG_MODE=cta timeout 900 python tools/diag_tucker.py C4 2 5 > gpurun_out/b_diag_cta.log 2>&1
timeout 300 python tools/sinr_once.py C4 16 > gpurun_out/b_once.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_sinr_launches.csv python tools/sinr_once.py C4 16 > gpurun_out/b_ncu1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_tucker_launches.csv python tools/tucker_once.py C4 16 2 > gpurun_out/b_ncu2.log 2>&1
