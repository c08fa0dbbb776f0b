"""Small driver for profiling K1 (and K3) on the C4 state: builds the
shallow-water level, then launches K1 `--launches` times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1511_03645_b200 import _lib, device, solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--launches", type=int, default=3)
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--variant", default="fast")
ap.add_argument("--flag", action="store_true")
ap.add_argument("--flag1", action="store_true", help="single-snapshot window")
ap.add_argument("--coast", action="store_true", help="C4 + 1500 m: coastline, wet/dry kernel")
ap.add_argument("--phys-in", action="store_true", help="the bench's launch (fills its input's physical ghosts)")
a = ap.parse_args()
bench.N = a.n
h, p, eq, bc, dt = bench.build_c4(a.n, land=1500.0 if a.coast else 0.0)
if a.coast:
    bc = solver.BoundarySpec("wall", "wall", "wall", "wall")
st = solver.store_of(p)
st.sync_in()
var = _lib.VARIANT_FAST if a.variant == "fast" else _lib.VARIANT_EXACT
solver.advance_uniform(p, eq, bc, (a.n, a.n), dt, 2, "MC", var)
torch.cuda.synchronize()
times = []
for _ in range(a.launches):
    out = st._free(st.cur, -1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    device.launch_step(st, dt, eq, "MC", var, out, phys_in=(bc, eq, (a.n, a.n)) if a.phys_in else None)
    e1.record()
    st.ghost_src = st.cur
    st.cur = out
    times.append((e0, e1))
torch.cuda.synchronize()
ms = [x.elapsed_time(y) for x, y in times]
print("k1 ms:", [round(v, 4) for v in ms], "median", round(sorted(ms)[len(ms) // 2], 4), os.environ.get("ADJAMR_LIB", "default"))
if a.flag or a.flag1:
    ring = bench.adjoint_ring(41)
    device.launch_flag(st, ring, (1024, 1024), (0.0, 0.0), bench.L / 1024, bench.L / 1024, (0.0, 0.0),
                       bench.L / a.n, bench.L / a.n, [20] if a.flag1 else list(range(20, 41)), 1e-4)
    torch.cuda.synchronize()
print("ok")
