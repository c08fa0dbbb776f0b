"""A/B of one library build (ADJAMR_LIB=...): C4 step + K1 alone, C3 step + K1
alone, C5 coarse step, and the FAST-vs-EXACT norm-relative difference after
``--err-steps`` steps on C4 and C3.  One JSON line."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1511_03645_b200 import _lib, solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--err-steps", type=int, default=20)
ap.add_argument("--no-c5", action="store_true")
a = ap.parse_args()
res = {"lib": os.path.basename(os.environ.get("ADJAMR_LIB", "default"))}


def timed_uniform(p, eq, bc, shape, dt, steps):
    solver.advance_uniform(p, eq, bc, shape, dt, 4, "MC", _lib.VARIANT_FAST)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    solver.advance_uniform(p, eq, bc, shape, dt, steps, "MC", _lib.VARIANT_FAST)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def err(build, shape):
    outs = []
    for var in (_lib.VARIANT_EXACT, _lib.VARIANT_FAST):
        h, p, eq, bc, dt = build()
        solver.advance_uniform(p, eq, bc, shape, dt, a.err_steps, "MC", var)
        outs.append(p.interior().copy())
    e, f = outs
    return max(float(np.max(np.abs(f[c] - e[c])) / max(np.max(np.abs(e[c])), 1e-300)) for c in range(e.shape[0]))


n = bench.N
h, p, eq, bc, dt = bench.build_c4(n)
res["c4_step_ms"] = round(timed_uniform(p, eq, bc, (n, n), dt, a.steps), 5)
res["c4_k1_ms"] = round(bench.k1_alone_ms(solver.store_of(p), dt, eq, _lib.VARIANT_FAST, 10, phys_in=(bc, eq, (n, n))), 5)
del h, p
h, p, eq, bc, dt = bench.build_c3(2048)
res["c3_step_ms"] = round(timed_uniform(p, eq, bc, (2048, 2048), dt, a.steps), 5)
res["c3_k1_ms"] = round(bench.k1_alone_ms(solver.store_of(p), dt, eq, _lib.VARIANT_FAST, 10,
                                          phys_in=(bc, eq, (2048, 2048))), 5)
del h, p
torch.cuda.empty_cache()
if not a.no_c5:
    res["c5_ms"] = round(bench.bench_c5(20, 3, _lib.VARIANT_FAST)["ms_per_coarse_step"], 5)
res["c4_err"] = err(lambda: bench.build_c4(n), (n, n))
res["c3_err"] = err(lambda: bench.build_c3(2048), (2048, 2048))
print(json.dumps(res), flush=True)
