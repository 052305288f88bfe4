for m in jacobi warp cta; do echo "mode=$m"; GWT_EIG_MODE=$m timeout 200 python tools/eig_probe.py > gpurun_out/ep_$m.log 2>&1; grep -E "batch|Error" gpurun_out/ep_$m.log; done
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['tucker']['ms_per_solve'], d['tucker']['stage_ms'])"
