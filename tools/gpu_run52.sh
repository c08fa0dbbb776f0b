mkdir -p gpurun_out
rm -f gpurun_out/k3ab.log
for v in 0 0; do
  ADJAMR_K3_ROWAL=$v python bench.py --no-c5 --no-cpu-baseline --steps 5 > gpurun_out/bench52_$v.log 2>&1
  tail -1 gpurun_out/bench52_$v.log | V=$v python tools/flagline.py >> gpurun_out/k3ab.log
done
python -m pytest tests -q -m gpu -x > gpurun_out/pytest52.log 2>&1
echo done
