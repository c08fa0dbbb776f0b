import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, adjoint, amr, device
stats = {"zeros_ms": 0.0, "zeros_n": 0, "idle_wait_ms": 0.0}
_orig = torch.zeros
def timed_zeros(*a, **k):
    if k.get("device") == "cuda":
        t0 = time.perf_counter(); torch.cuda.synchronize(); t1 = time.perf_counter()
        r = _orig(*a, **k)
        t2 = time.perf_counter()
        stats["idle_wait_ms"] += 1e3 * (t1 - t0); stats["zeros_ms"] += 1e3 * (t2 - t1); stats["zeros_n"] += 1
        return r
    return _orig(*a, **k)
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
steps = 13
T = steps * dt
window = adjoint.TimeWindow(0.0, T)
store = adjoint.solve_adjoint(eq, ctx.boundary, adjoint.FunctionalSpec("box", (0.6, 0.7, 0.3, 0.4), (1.0, 0.0, 0.0)),
                              window, (0.0, 1.0), (0.0, 1.0), (1024, 1024), t0=0.0, dt_snap=T / 64, keep_on_device=True)
ctx.strategy = adjoint.AdjointFlagging(store, window, 1e-9, time_interp=True)
ctx.regrid_interval = 4
ctx.max_patch_edge = 64
amr.advance_hierarchy(h, 1, dt, ctx)
torch.cuda.synchronize()
torch.zeros = timed_zeros
t0 = time.perf_counter()
for k in range(steps - 2):
    amr.advance_hierarchy(h, 1, dt, ctx)
torch.cuda.synchronize()
print("total ms", 1e3 * (time.perf_counter() - t0), stats)
