mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest63.log 2>&1
python tools/diag_phases.py > gpurun_out/diag_phases63.log 2>&1
echo done
