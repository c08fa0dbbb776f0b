mkdir -p gpurun_out
s=$(date +%s); python bench.py > gpurun_out/bench58.log 2> gpurun_out/bench58.err; e=$(date +%s); echo "bench wall $((e-s)) s" > gpurun_out/bench58.time
echo done
