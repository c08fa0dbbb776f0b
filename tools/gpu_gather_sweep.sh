# C5 graph time per coarse step for gather variants: entries per thread (ADJAMR_GATHER_U) x experiment libraries
T=$1; shift
mkdir -p gpurun_out/$T
for L in default "$@"; do
  for U in 1 2 4; do
    if [ "$L" = default ]; then unset ADJAMR_LIB; else export ADJAMR_LIB=tools/exp/lib_$L.so; fi
    echo "lib=$L U=$U" >> gpurun_out/$T/sweep.txt
    ADJAMR_GATHER_U=$U python tools/c5_graph_time.py 2>&1 | tail -2 >> gpurun_out/$T/sweep.txt
  done
done
cat gpurun_out/$T/sweep.txt
