# K3 row kernel: cells per lane / run length / unroll variants
mkdir -p gpurun_out/r72
for v in base u2 p8 nc2 nc2r32 nc2r8 nc2u2 base nc2; do
  if [ $v = base ]; then L=; else L=tools/exp/lib_$v.so; fi
  ADJAMR_LIB=$L V=$v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c5 --c5-full 0 2>/dev/null | V=$v python tools/flagline.py >> gpurun_out/r72/ab.txt
done
echo done
