mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest38.log 2>&1
timeout 900 python tools/prof_regrid.py > gpurun_out/prof_regrid38.log 2>&1
echo done
