mkdir -p gpurun_out
./tools/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
python tools/prof_k1.py --launches 5 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 2 -c 1 -o gpurun_out/k1_r1 python tools/prof_k1.py --launches 3 > gpurun_out/ncu_k1.log 2>&1
echo done
