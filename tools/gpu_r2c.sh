mkdir -p gpurun_out/r2c
python -m pytest tests/test_gpu_job_fill.py tests/test_gpu_amr.py tests/test_gpu_fused_restrict.py -x -q > gpurun_out/r2c/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2c/pytest.log
python tools/c5_graph_time.py > gpurun_out/r2c/c5_on.log 2>&1
ADJAMR_JOB_FILL=0 python tools/c5_graph_time.py > gpurun_out/r2c/c5_off.log 2>&1
tail -5 gpurun_out/r2c/pytest.log; cat gpurun_out/r2c/c5_on.log gpurun_out/r2c/c5_off.log
