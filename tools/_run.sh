for v in "GWT_REBUILD_GSMEM=1" "GWT_REBUILD_GSMEM=0" "GWT_REBUILD_GSMEM=1" "GWT_REBUILD_GSMEM=0"; do echo "$v $(env GWT_SINR_DEV_LANES=1 $v timeout 120 python tools/sinr_time.py C2 100 | tail -1) | 2L $(env $v timeout 120 python tools/sinr_time.py C2 100 | tail -1 | cut -c1-40)"; done
for c in C3 C5; do echo "$c $(GWT_SINR_DEV_LANES=1 timeout 200 python tools/sinr_time.py $c 3 | tail -1)"; done
