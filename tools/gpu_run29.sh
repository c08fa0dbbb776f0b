mkdir -p gpurun_out
rm -f gpurun_out/sweep29.log
for v in base mb4 w1r144 w1r136 w1r128 w2r144 w2m7 base w1r144; do
  ADJAMR_LIB=tools/exp/lib_$v.so timeout 300 python tools/prof_k1.py --launches 20 2>&1 | grep "k1 ms" >> gpurun_out/sweep29.log
done
echo done
