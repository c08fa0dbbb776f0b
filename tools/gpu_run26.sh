mkdir -p gpurun_out
timeout 900 python tools/c5_full.py 9 > gpurun_out/c5_full.log 2>&1
echo done
