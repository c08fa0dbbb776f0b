mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest48.log 2>&1
python tools/prof_k1.py --launches 20 > gpurun_out/k1_48.log 2>&1
python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench48.log 2>&1
echo done
