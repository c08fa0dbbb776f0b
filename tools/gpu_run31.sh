mkdir -p gpurun_out
python tools/c5_one_step.py 2 > gpurun_out/c5_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_rects -s 6 -c 2 -o gpurun_out/k2_rects_c5 -f python tools/c5_one_step.py 2 > gpurun_out/ncu31a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 4 -c 2 -o gpurun_out/k1_c5 -f python tools/c5_one_step.py 2 > gpurun_out/ncu31b.log 2>&1
echo done
