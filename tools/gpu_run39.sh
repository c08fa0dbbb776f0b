mkdir -p gpurun_out
python -m pytest tests/test_gpu_output.py -q -x > gpurun_out/pytest39.log 2>&1
python -m pytest tests -q -m gpu > gpurun_out/pytest39_all.log 2>&1
echo done
