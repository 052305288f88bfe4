for cfg in "16 128" "16 256" "16 64" "8 64" "8 128" "8 256"; do set -- $cfg; GWT_RG_FT=$1 GWT_RG_WG=$2 timeout 120 python bench.py --no-cpu-baseline --steps 100 --warmup 5 > gpurun_out/sw_$1_$2.log 2>&1; python -c "
import json,sys
d=json.loads(open('gpurun_out/sw_$1_$2.log').read().strip().splitlines()[-1]); print('FT=$1 WG=$2', round(d['ms_per_step'],4), d['roofline']['stage_ms'])
"; done; GWT_SINR_PATH=generic timeout 120 python bench.py --no-cpu-baseline --steps 100 --warmup 5 > gpurun_out/sw_gen.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/sw_gen.log').read().strip().splitlines()[-1]); print('generic', round(d['ms_per_step'],4), d['roofline']['stage_ms'])"
