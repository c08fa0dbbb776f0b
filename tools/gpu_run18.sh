mkdir -p gpurun_out
python tools/prof_k1.py --launches 1 --flag > gpurun_out/prof_flag_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k3_flag -c 1 -o gpurun_out/k3_r1 python tools/prof_k1.py --launches 1 --flag > gpurun_out/ncu_k3.log 2>&1
echo done
