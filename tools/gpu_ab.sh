# A/B on the GPU box: tools/ab.py for the working-tree library and each tools/exp/lib_*.so given.
# Usage: bash tools/gpu_ab.sh <tag> [lib names...]   (each run twice, interleaved)
T=$1; shift
mkdir -p gpurun_out/$T
for rep in 1 2; do
  python tools/ab.py "${AB_ARGS[@]}" >> gpurun_out/$T/ab.txt 2>&1
  for L in "$@"; do ADJAMR_LIB=tools/exp/lib_$L.so python tools/ab.py >> gpurun_out/$T/ab.txt 2>&1; done
done
cat gpurun_out/$T/ab.txt | grep lib
