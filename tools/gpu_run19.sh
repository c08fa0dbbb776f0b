mkdir -p gpurun_out
python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-c5 > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-c5 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_k1.py --launches 3 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 2 -c 1 -o gpurun_out/r01_k1_c4 python tools/prof_k1.py --launches 3 > gpurun_out/ncu_k1.log 2>&1
python tools/prof_k1.py --launches 1 --flag > gpurun_out/prof_flag_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k3_flag -c 1 -o gpurun_out/r01_k3_c4 python tools/prof_k1.py --launches 1 --flag > gpurun_out/ncu_k3.log 2>&1
echo done
