mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "amr or adjoint" > gpurun_out/pytest_amr.log 2>&1
echo done
