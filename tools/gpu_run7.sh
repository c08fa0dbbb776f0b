mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ghost_restrict.py -q > gpurun_out/pytest_gr.log 2>&1
timeout 600 python tools/diag_adjoint.py > gpurun_out/diag_adjoint.log 2>&1
echo done
