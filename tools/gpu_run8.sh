mkdir -p gpurun_out
timeout 600 python tools/diag_amr.py > gpurun_out/diag_amr.log 2>&1
timeout 600 python -m pytest tests/test_gpu_amr.py -q -k solve_adjoint > gpurun_out/pytest_sa.log 2>&1
echo done
