mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest35.log 2>&1
python tools/c5_graph_time.py > gpurun_out/c5_graph35.log 2>&1
ADJAMR_PDL=0 python tools/c5_graph_time.py > gpurun_out/c5_graph35_nopdl.log 2>&1
python tools/prof_k1.py --launches 20 > gpurun_out/k1_35.log 2>&1
echo done
