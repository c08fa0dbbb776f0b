mkdir -p gpurun_out/r64
python bench.py > gpurun_out/r64/bench.log 2> gpurun_out/r64/bench.err
python bench.py --impl reference > gpurun_out/r64/ref.log 2> gpurun_out/r64/ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r64/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 > gpurun_out/r64/ncu_list.log 2>&1
python tools/c5_graph_time.py > gpurun_out/r64/c5_graph.log 2>&1
NCU_ONE=1 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/r64/launches_c5_warm.csv python tools/c5_graph_time.py > gpurun_out/r64/ncu_c5list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 2 -c 1 -o gpurun_out/r64/k1_c4 -f python tools/prof_k1.py --launches 3 > gpurun_out/r64/ncu_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 4 -c 1 -o gpurun_out/r64/k1_c5 -f python tools/c5_one_step.py 2 > gpurun_out/r64/ncu_k1c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k3_ -c 1 -o gpurun_out/r64/k3_c4_single -f python tools/prof_k1.py --launches 1 --flag1 > gpurun_out/r64/ncu_k3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k3_pair -c 1 -o gpurun_out/r64/k3_c4_pair -f python tools/prof_k1.py --launches 1 --flag > gpurun_out/r64/ncu_k3p.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_gather -s 20 -c 1 -o gpurun_out/r64/gather_c5 -f python tools/c5_one_step.py 3 > gpurun_out/r64/ncu_g.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k4_cells -s 3 -c 1 -o gpurun_out/r64/k4_c5 -f python tools/c5_one_step.py 3 > gpurun_out/r64/ncu_k4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k5_flags -c 1 -o gpurun_out/r64/k5 -f python tools/prof_regrid.py > gpurun_out/r64/ncu_k5.log 2>&1
echo done
