mkdir -p gpurun_out
python tools/diag_uniform.py > gpurun_out/diag_uniform.log 2>&1
echo done
