mkdir -p gpurun_out
for v in base w1r168 w1r152 w1r144 w1r136 w2r152 base; do
  ADJAMR_LIB=tools/exp/lib_$v.so timeout 300 python tools/prof_k1.py --launches 20 2>&1 | grep "k1 ms" >> gpurun_out/sweep28.log
done
echo done
