mkdir -p gpurun_out
rm -f gpurun_out/sweep29.log
for v in base c1 base c1; do
  ADJAMR_LIB=tools/exp/lib_$v.so timeout 300 python tools/prof_k1.py --launches 20 2>&1 | grep "k1 ms" >> gpurun_out/sweep29.log
done
echo done
