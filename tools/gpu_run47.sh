mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest47.log 2>&1
python bench.py --no-c5 --no-cpu-baseline --steps 10 > gpurun_out/bench47.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k3_ -c 1 -o gpurun_out/k3t_c4 -f python tools/prof_k1.py --launches 1 --flag > gpurun_out/ncu47.log 2>&1
echo done
