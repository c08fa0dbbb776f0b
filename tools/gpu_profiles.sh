# Round-end evidence on the GPU box, in three parts so each call's gpurun_out/ stays under 64 MiB:
#   bash tools/gpu_profiles.sh bench   -- GPU tests, bench line, reference arm, launch lists
#   bash tools/gpu_profiles.sh c4      -- ncu --set full: K1 (C4), K3 single (k3_rowp), K3 full span (k3_quad)
#   bash tools/gpu_profiles.sh c5      -- ncu --set full: K3 C3 (k3_direct), K1 (C5), gather, K4
# Each profiled command first runs clean without ncu.
set -x
O=gpurun_out/prof
mkdir -p $O
case "$1" in
bench)
  python -m pytest tests -m gpu -x -q > $O/tests.txt 2>&1; tail -1 $O/tests.txt
  python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
  python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
  python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.json 2> $O/ref.err; echo "ref exit $?"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 > $O/ncu_list.log 2>&1
  python tools/c5_graph_time.py > $O/c5_graph.log 2>&1
  NCU_ONE=1 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/launches_c5_warm.csv python tools/c5_graph_time.py > $O/ncu_c5list.log 2>&1
  ;;
c4)
  python tools/prof_k1.py --launches 3 > $O/prof_k1.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 2 -c 1 -o $O/k1_c4 -f python tools/prof_k1.py --launches 3 > $O/ncu_k1.log 2>&1
  python tools/prof_k1.py --launches 1 --flag1 > $O/prof_k3.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k3_rowp -c 1 -o $O/k3_c4_single -f python tools/prof_k1.py --launches 1 --flag1 > $O/ncu_k3.log 2>&1
  python tools/prof_k1.py --launches 1 --flag > $O/prof_k3q.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k3_quad -c 1 -o $O/k3_c4_span -f python tools/prof_k1.py --launches 1 --flag > $O/ncu_k3q.log 2>&1
  ;;
c5)
  python tools/prof_c3.py 1 flag > $O/prof_c3.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k3_direct -c 1 -o $O/k3_c3_direct -f python tools/prof_c3.py 1 flag > $O/ncu_k3d.log 2>&1
  python tools/c5_one_step.py 3 > $O/c5_one.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 4 -c 1 -o $O/k1_c5 -f python tools/c5_one_step.py 2 > $O/ncu_k1c5.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k2_gather -s 20 -c 1 -o $O/gather_c5 -f python tools/c5_one_step.py 3 > $O/ncu_g.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k4_cells -s 1 -c 1 -o $O/k4_c5 -f python tools/c5_one_step.py 3 > $O/ncu_k4.log 2>&1
  ;;
esac
ls -la $O
echo done
