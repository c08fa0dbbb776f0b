mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1
python tools/prof_k1.py --launches 10 > gpurun_out/prof_k1.log 2>&1
ADJAMR_K1_ROWS=1 python tools/prof_k1.py --launches 10 > gpurun_out/prof_k1_rows1.log 2>&1
echo done
