# full GPU suite + bench + K3 row-kernel capture
mkdir -p gpurun_out/r73
python -m pytest tests -q -m gpu -x > gpurun_out/r73/tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r73/tests.log
python bench.py > gpurun_out/r73/bench.log 2> gpurun_out/r73/bench.err
ncu --set full --clock-control none --import-source on -k regex:k3_ -c 1 -o gpurun_out/r73/k3_c4_single -f python tools/prof_k1.py --launches 1 --flag1 > gpurun_out/r73/ncu_k3.log 2>&1
echo done
