# Round-2 evidence: ncu --set full of the pruned K3 full-span pipeline (C4) and of K1 on C5
# (one launch each), each command first run clean without ncu.
set -x
O=gpurun_out/prof2
mkdir -p $O
python tools/prof_k1.py --launches 1 --flag > $O/prof_k3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k3_bound|k3_quad_list|k3_envelope" -c 4 -o $O/k3_pruned -f python tools/prof_k1.py --launches 1 --flag > $O/ncu_k3.log 2>&1
python tools/c5_one_step.py 2 > $O/c5_one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 4 -c 1 -o $O/k1_c5 -f python tools/c5_one_step.py 2 > $O/ncu_k1c5.log 2>&1
ls -la $O
