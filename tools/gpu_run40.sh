mkdir -p gpurun_out/r40
python bench.py > gpurun_out/r40/bench.log 2> gpurun_out/r40/bench.err
python bench.py --impl reference > gpurun_out/r40/ref.log 2> gpurun_out/r40/ref.err
python bench.py --c5-full 9 --no-cpu-baseline --steps 10 > gpurun_out/r40/c5full.log 2> gpurun_out/r40/c5full.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r40/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r40/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 2 -c 1 -o gpurun_out/r40/k1_c4 -f python tools/prof_k1.py --launches 3 > gpurun_out/r40/ncu_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_gather -s 20 -c 1 -o gpurun_out/r40/gather_c5 -f python tools/c5_one_step.py 3 > gpurun_out/r40/ncu_g.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k4_cells -s 3 -c 1 -o gpurun_out/r40/k4_c5 -f python tools/c5_one_step.py 3 > gpurun_out/r40/ncu_k4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k3_flag -c 1 -o gpurun_out/r40/k3_c4 -f python tools/prof_k1.py --launches 1 --flag > gpurun_out/r40/ncu_k3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k5_flags -c 1 -o gpurun_out/r40/k5 -f python tools/prof_regrid.py > gpurun_out/r40/ncu_k5.log 2>&1
echo done
