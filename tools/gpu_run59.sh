mkdir -p gpurun_out
timeout 900 python tools/prof_c5_full.py 13 > gpurun_out/prof_c5_full59.log 2>&1
echo done
