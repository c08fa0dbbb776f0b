mkdir -p gpurun_out
timeout 900 python tools/prof_regrid.py > gpurun_out/prof_regrid37.log 2>&1
echo done
