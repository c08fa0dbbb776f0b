# Iteration check on the GPU box: the GPU tests, then the default bench line.
# Usage: bash tools/gpu_iter.sh <tag>
T=${1:-iter}
mkdir -p gpurun_out/$T
python -m pytest tests -m gpu -x -q > gpurun_out/$T/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$T/pytest.log
python bench.py > gpurun_out/$T/bench.log 2> gpurun_out/$T/bench.err
tail -3 gpurun_out/$T/pytest.log
python - <<'PY' "$T"
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}/bench.log").read().strip().splitlines()[-1])
r = d["roofline"]
print("C4 step ms", d["ms_per_step"], "K1 ms", r["kernel_ms"], "frac", round(r["frac"], 4))
print("C5 ms/coarse", d["c5_batched_patches"]["ms_per_coarse_step"], "C3 step", d["c3_heterogeneous_acoustics"]["ms_per_step"],
      "C3 K1", d["c3_heterogeneous_acoustics"]["k1_ms"])
print("flag single", d["flagging"]["kernel_ms"], "full", d["flagging"]["full_span"]["kernel_ms"], "fast", d["flagging"]["full_span_fast"]["kernel_ms"])
print("clocks", d["clocks"])
PY
