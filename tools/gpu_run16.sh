mkdir -p gpurun_out
python tools/c5_one_step.py 2 > gpurun_out/c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 14 -c 1 -o gpurun_out/k1_c5 python tools/c5_one_step.py 2 > gpurun_out/c5_ncu_full.log 2>&1
python tools/c5_one_step.py 2 > gpurun_out/c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_rects -s 14 -c 1 -o gpurun_out/k2_c5 python tools/c5_one_step.py 2 > gpurun_out/c5_ncu_full2.log 2>&1
echo done
