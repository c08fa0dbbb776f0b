mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest42.log 2>&1
timeout 900 python tools/prof_c5_full.py 9 > gpurun_out/prof_c5_full42.log 2>&1
echo done
