mkdir -p gpurun_out
GWT_PG_SMALL=1 timeout 300 python tools/sinr_once.py C4 4 > gpurun_out/k_once_small.log 2>&1; echo "rc $?" >> gpurun_out/k_once_small.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/sinr_once.py C4 4 > gpurun_out/k_once_def.log 2>&1; echo "rc $?" >> gpurun_out/k_once_def.log
