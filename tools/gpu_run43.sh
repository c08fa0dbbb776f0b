mkdir -p gpurun_out
python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/pytest43.log 2>&1
python bench.py --no-c5 --no-cpu-baseline --steps 10 > gpurun_out/bench43.log 2>&1
echo done
