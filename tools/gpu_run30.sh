mkdir -p gpurun_out
python tools/c5_one_step.py 3 > gpurun_out/c5_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_r30.csv python tools/c5_one_step.py 3 > gpurun_out/ncu30.log 2>&1
python bench.py --steps 10 --warmup 4 > gpurun_out/bench30.log 2>&1
echo done
