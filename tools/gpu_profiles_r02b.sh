# Round-2 evidence (second session): GPU tests, smoke, bench line, reference arm, ncu --set full of
# K1 on C4 (the bench's launch) and on the C4 coastline (wet/dry instantiation), C5 warm launch list.
# Each profiled command first runs clean without ncu.
# Two calls (each call's gpurun_out/ must stay under 64 MiB): bash tools/gpu_profiles_r02b.sh a|b
set -x
O=gpurun_out/prof_r02b
mkdir -p $O
if [ "$1" = a ]; then
python -m pytest tests -m gpu -x -q > $O/tests.txt 2>&1; tail -1 $O/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
python bench.py --impl reference --steps 3 --warmup 3 > $O/ref.json 2> $O/ref.err; echo "ref exit $?"
python tools/prof_k1.py --launches 3 --phys-in > $O/prof_k1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 2 -c 1 -o $O/k1_c4 -f python tools/prof_k1.py --launches 3 --phys-in > $O/ncu_k1.log 2>&1
fi
if [ "$1" = b ]; then
python tools/prof_k1.py --launches 3 --phys-in --coast > $O/prof_k1wd.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 2 -c 1 -o $O/k1_coast -f python tools/prof_k1.py --launches 3 --phys-in --coast > $O/ncu_k1wd.log 2>&1
python tools/c5_graph_time.py > $O/c5_graph.log 2>&1 && \
NCU_ONE=1 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/launches_c5_warm.csv python tools/c5_graph_time.py > $O/ncu_c5list.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 > $O/ncu_list.log 2>&1
fi
ls -la $O
