mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k2_gather -s 20 -c 3 -o gpurun_out/k2_gather_c5 -f python tools/c5_one_step.py 3 > gpurun_out/ncu34a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k4_restrict -s 3 -c 2 -o gpurun_out/k4_c5 -f python tools/c5_one_step.py 3 > gpurun_out/ncu34b.log 2>&1
echo done
