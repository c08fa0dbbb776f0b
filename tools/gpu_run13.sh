mkdir -p gpurun_out
timeout 600 python tools/prof_c5_host.py > gpurun_out/prof_c5_host.log 2>&1
echo done
