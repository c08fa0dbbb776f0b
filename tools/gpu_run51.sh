mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest51.log 2>&1
for v in 1 0 1 0; do ADJAMR_K3_ROWAL=$v python bench.py --no-c5 --no-cpu-baseline --steps 5 > gpurun_out/bench51_$v.log 2>&1; tail -1 gpurun_out/bench51_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); f=d['flagging']; print("rowal", "$v", f['value']/1e9, f['kernel_ms'], f['full_span']['value']/1e9, f['full_span']['kernel_ms'], f['flagged'])" >> gpurun_out/k3ab.log; done
ncu --set full --clock-control none --import-source on -k regex:k3_ -c 1 -o gpurun_out/k3p_c4 -f python tools/prof_k1.py --launches 1 --flag > gpurun_out/ncu51.log 2>&1
echo done
