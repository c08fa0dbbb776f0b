mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke50.log 2>&1
python bench.py > gpurun_out/bench50.log 2> gpurun_out/bench50.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref50.log 2>&1
echo done
