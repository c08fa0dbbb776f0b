mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest36.log 2>&1
python tools/c5_graph_time.py > gpurun_out/c5_graph36.log 2>&1
NCU_ONE=1 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_c5_warm36.csv python tools/c5_graph_time.py > gpurun_out/ncu36.log 2>&1
echo done
