mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_full.log 2>&1
echo done
