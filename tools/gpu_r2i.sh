mkdir -p gpurun_out/r2i
python -m pytest tests -m gpu -x -q > gpurun_out/r2i/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2i/pytest.log
python tools/kbench.py --no-k1 > gpurun_out/r2i/kb_on.log 2>&1
ADJAMR_FLAG_PRUNE=0 python tools/kbench.py --no-k1 > gpurun_out/r2i/kb_off.log 2>&1
python tools/c5_full.py 12 > gpurun_out/r2i/c5full.log 2>&1
tail -3 gpurun_out/r2i/pytest.log; cat gpurun_out/r2i/kb_on.log gpurun_out/r2i/kb_off.log; cut -c1-600 gpurun_out/r2i/c5full.log
