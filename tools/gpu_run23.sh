mkdir -p gpurun_out
python bench.py --steps 6 --warmup 4 --no-cpu-baseline --no-c5 > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k[1-4]_|k1_fast" --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 6 --warmup 4 --no-cpu-baseline --no-c5 > gpurun_out/ncu_launch.log 2>&1
python tools/c5_one_step.py 3 > gpurun_out/c5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k[1-4]_|k1_fast" --csv --log-file gpurun_out/launches_c5.csv python tools/c5_one_step.py 3 > gpurun_out/c5_ncu.log 2>&1
echo done
