mkdir -p gpurun_out
rm -f gpurun_out/k3ab.log
python -m pytest tests -q -m gpu -x > gpurun_out/pytest54.log 2>&1
for v in 1 0 1 0; do
  ADJAMR_K3_TILE=$v python bench.py --no-c5 --no-cpu-baseline --steps 5 > gpurun_out/bench54_$v.log 2>&1
  tail -1 gpurun_out/bench54_$v.log | V=$v python tools/flagline.py >> gpurun_out/k3ab.log
done
ncu --set full --clock-control none --import-source on -k regex:k3_ -c 1 -o gpurun_out/k3tile_c4 -f python tools/prof_k1.py --launches 1 --flag1 > gpurun_out/ncu54.log 2>&1
echo done
