mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest56.log 2>&1
python tools/c5_graph_time.py > gpurun_out/c5_graph56.log 2>&1
echo done
