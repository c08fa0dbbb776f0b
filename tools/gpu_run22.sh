mkdir -p gpurun_out
: > gpurun_out/variants.log
for v in base v1_finite v2_ky v3_g3 v4_ni256 v5_ni64 v6_all; do
  if [ "$v" = base ]; then L=paper_1511_03645_b200/libadjamr_b200.so; else L=tools/exp/lib_$v.so; fi
  echo "== $v" >> gpurun_out/variants.log
  ADJAMR_LIB=$L python tools/prof_k1.py --launches 10 >> gpurun_out/variants.log 2>&1
done
echo done
