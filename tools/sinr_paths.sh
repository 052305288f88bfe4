for pth in default generic; do
  if [ $pth = default ]; then unset GWT_SINR_PATH; else export GWT_SINR_PATH=$pth; fi
  timeout 120 python bench.py --no-cpu-baseline --steps 100 --warmup 5 > gpurun_out/sp_$pth.log 2>&1; echo "== $pth"; python tools/show_bench.py gpurun_out/sp_$pth.log | head -4
done
unset GWT_SINR_PATH
for ft in 2 4 8; do GWT_RG_FT=$ft timeout 120 python bench.py --no-cpu-baseline --steps 100 --warmup 5 > gpurun_out/sp_ft$ft.log 2>&1; echo "== FT=$ft $(python tools/show_bench.py gpurun_out/sp_ft$ft.log | head -1)"; done
