mkdir -p gpurun_out
python tools/prof_k1.py --launches 1 --flag1 > gpurun_out/k3once.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k3_ -c 1 -o gpurun_out/k3t1_c4 -f python tools/prof_k1.py --launches 1 --flag1 > gpurun_out/ncu53.log 2>&1
echo done
