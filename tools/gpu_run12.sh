mkdir -p gpurun_out
timeout 600 python tools/diag_graph.py > gpurun_out/diag_graph.log 2>&1
echo done
