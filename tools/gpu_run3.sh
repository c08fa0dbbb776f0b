mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1
python tools/prof_k1.py --launches 8 > gpurun_out/prof_plain.log 2>&1
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
python tools/prof_k1.py --launches 3 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 2 -c 1 -o gpurun_out/k1_r2 python tools/prof_k1.py --launches 3 > gpurun_out/ncu_k1.log 2>&1
echo done
