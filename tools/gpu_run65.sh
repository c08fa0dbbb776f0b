mkdir -p gpurun_out
rm -f gpurun_out/c4ab.log
python -m pytest tests -q -m gpu -x > gpurun_out/pytest65.log 2>&1
for v in 1 0 1 0; do ADJAMR_PDL=$v python bench.py --no-c5 --no-cpu-baseline --steps 50 > gpurun_out/b65_$v.log 2>&1; tail -1 gpurun_out/b65_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl', '$v', d['value']/1e9, d['ms_per_step'])" >> gpurun_out/c4ab.log; done
echo done
