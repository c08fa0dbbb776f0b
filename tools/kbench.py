"""A/B timing of the C4 kernels for experiment libraries (ADJAMR_LIB=...):
K1 alone (median of --launches), K3 single-snapshot and full-span windows.
Prints one line per run: lib, K1 ms, K3 single ms, K3 full-span ms, flagged."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1511_03645_b200 import _lib, adjoint, device, solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--launches", type=int, default=21)
ap.add_argument("--no-k1", action="store_true")
ap.add_argument("--no-flag", action="store_true")
a = ap.parse_args()
n = bench.N
h, p, eq, bc, dt = bench.build_c4(n)
st = solver.store_of(p)
st.sync_in()
var = _lib.VARIANT_FAST
solver.advance_uniform(p, eq, bc, (n, n), dt, 2, "MC", var)
torch.cuda.synchronize()
res = {"lib": os.path.basename(os.environ.get("ADJAMR_LIB", "default"))}
if not a.no_k1:
    ms = []
    for _ in range(a.launches):
        out = st._free(st.cur, -1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        device.launch_step(st, dt, eq, "MC", var, out)
        e1.record()
        st.ghost_src = st.cur
        st.cur = out
        ms.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(x.elapsed_time(y) for x, y in ms)
    res["k1_ms"] = round(v[len(v) // 2], 4)
    res["k1_min"] = round(v[0], 4)
if not a.no_flag:
    ring = bench.adjoint_ring(41)
    times = np.linspace(0.0, bench.T_STEPS * dt, 41)
    t = 150 * dt
    for label, ts in (("single", bench.T_STEPS * dt), ("span", 0.0)):
        idx = adjoint.window_indices(t, adjoint.TimeWindow(ts, bench.T_STEPS * dt), times)
        args = (st, ring, (1024, 1024), (0.0, 0.0), bench.L / 1024, bench.L / 1024, (0.0, 0.0), bench.L / n,
                bench.L / n, idx, bench.FLAG_TOL)
        device.launch_flag(*args)
        torch.cuda.synchronize()
        reps = 10
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph, stream=side):
                for _ in range(reps):
                    _, counts, _, _ = device.launch_flag(*args)
        torch.cuda.current_stream().wait_stream(side)
        gph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gph.replay()
        e1.record()
        torch.cuda.synchronize()
        res[f"k3_{label}_ms"] = round(e0.elapsed_time(e1) / reps, 4)
        res[f"k3_{label}_flagged"] = int(counts[0].item())
print(res, flush=True)
