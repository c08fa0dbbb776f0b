mkdir -p gpurun_out
python tools/c5_one_step.py 3 > gpurun_out/c5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/c5_one_step.py 3 > gpurun_out/c5_ncu.log 2>&1
echo done
