mkdir -p gpurun_out
python tools/prof_c3.py 6 > gpurun_out/prof_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 2 -c 1 -o gpurun_out/r01_k1_c3 python tools/prof_c3.py 3 > gpurun_out/ncu_c3.log 2>&1
echo done
