mkdir -p gpurun_out/r2d
python -m pytest tests/test_gpu_job_fill.py -x -q > gpurun_out/r2d/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2d/pytest.log
python tools/c5_graph_time.py > gpurun_out/r2d/c5_on.log 2>&1 && \
NCU_ONE=1 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/r2d/l_on.csv python tools/c5_graph_time.py > gpurun_out/r2d/ncu_on.log 2>&1
NCU_ONE=1 ADJAMR_JOB_FILL=0 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/r2d/l_off.csv python tools/c5_graph_time.py > gpurun_out/r2d/ncu_off.log 2>&1
tail -3 gpurun_out/r2d/pytest.log; cat gpurun_out/r2d/c5_on.log
