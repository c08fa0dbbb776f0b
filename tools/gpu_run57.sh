mkdir -p gpurun_out
python -m pytest tests/test_gpu_ghost_plan.py tests/test_gpu_amr.py -q -x > gpurun_out/pytest57.log 2>&1
for u in 1 2 4 1 2 4; do echo "U=$u" >> gpurun_out/c5_57.log; ADJAMR_GATHER_U=$u python tools/c5_graph_time.py 2>&1 | tail -1 >> gpurun_out/c5_57.log; done
echo done
