mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sinr_real.py C4 1 1 1 > gpurun_out/r7g_memcheck.log 2>&1; echo "rc $?" >> gpurun_out/r7g_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sinr_real.py C3 1 1 1 > gpurun_out/r7g_racecheck.log 2>&1; echo "rc $?" >> gpurun_out/r7g_racecheck.log
