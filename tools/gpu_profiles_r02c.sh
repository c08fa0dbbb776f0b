# Round-2 evidence (last session): GPU tests, smoke, bench line, reference arm, ncu --set full of
# K1 on C4 (the bench's launch), on C3 (per-job materials) and on the C5 sweep (invariant-material
# instantiation) with its gather, C5 warm launch list, bench launch list.
# Each profiled command first runs clean without ncu.  The reports stay on the box (68 MB each with
# the library's source): their summaries (tools/ncu_summary.py, ncu_stall_lines.py) come back.
# Calls: bash tools/gpu_profiles_r02c.sh a|b|c
set -x
O=gpurun_out/prof_r02c
R=/tmp/ncu_r02c
mkdir -p $O $R
summ() { python tools/ncu_summary.py $R/$1.ncu-rep > $O/$1_summary.txt 2>&1; python tools/ncu_stall_lines.py $R/$1.ncu-rep 14 > $O/$1_stalls.txt 2>&1; }
if [ "$1" = a ]; then
python -m pytest tests -m gpu -x -q > $O/tests.txt 2>&1; tail -1 $O/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
python bench.py --impl reference --steps 3 --warmup 3 > $O/ref.json 2> $O/ref.err; echo "ref exit $?"
fi
if [ "$1" = b ]; then
python tools/prof_k1.py --launches 3 --phys-in > $O/prof_k1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 2 -c 1 -o $R/k1_c4 -f python tools/prof_k1.py --launches 3 --phys-in > $O/ncu_k1.log 2>&1
summ k1_c4
python tools/prof_c3.py 3 physin > $O/prof_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 4 -c 1 -o $R/k1_c3 -f python tools/prof_c3.py 3 physin > $O/ncu_k1c3.log 2>&1
summ k1_c3
fi
if [ "$1" = c ] || [ "$1" = c1 ]; then
python tools/c5_one_step.py 3 > $O/c5_one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 26 -c 1 -o $R/k1_c5 -f python tools/c5_one_step.py 3 > $O/ncu_k1c5.log 2>&1
summ k1_c5
ncu --set full --clock-control none --cache-control none --import-source on -k regex:k2_gather -s 30 -c 1 -o $R/gather_c5 -f python tools/c5_one_step.py 3 > $O/ncu_gc5.log 2>&1
summ gather_c5
fi
if [ "$1" = c ]; then
python tools/c5_graph_time.py > $O/c5_graph.log 2>&1 && \
NCU_ONE=1 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/launches_c5_warm.csv python tools/c5_graph_time.py > $O/ncu_c5list.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 > $O/ncu_list.log 2>&1
fi
ls -la $O; du -sh gpurun_out
