"""cProfile of the C5 full workflow with caller tables for the hottest built-ins
(numpy.array, Tensor.to, ...) and a per-regrid phase split."""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, adjoint, amr

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 13
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
T = steps * dt
window = adjoint.TimeWindow(0.0, T)
store = adjoint.solve_adjoint(eq, ctx.boundary, adjoint.FunctionalSpec("box", (0.6, 0.7, 0.3, 0.4), (1.0, 0.0, 0.0)),
                              window, (0.0, 1.0), (0.0, 1.0), (1024, 1024), t0=0.0, dt_snap=T / 64,
                              keep_on_device=True)
ctx.strategy = adjoint.AdjointFlagging(store, window, 1e-9, time_interp=True)
ctx.regrid_interval = 4
ctx.max_patch_edge = 64
torch.cuda.synchronize()
pr = cProfile.Profile()
times = []
for step in range(steps):
    t0 = time.perf_counter()
    nreg = len(ctx.flagged_per_regrid)
    if step >= 1:
        pr.enable()
    amr.advance_hierarchy(h, 1, dt, ctx)
    torch.cuda.synchronize()
    pr.disable()
    times.append((round(1e3 * (time.perf_counter() - t0), 2), len(ctx.flagged_per_regrid) > nreg))
print("step ms (regrid?)", times)
print("patches", [len(h.patches(l)) for l in (1, 2, 3)])
st = pstats.Stats(pr)
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(70)
print(s.getvalue()[:16000])
for pat in ("numpy.array", "method 'to'", "repeat_interleave", "ufunc", "torch.zeros", "cumsum", "astype", "repeat' of"):
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_callers(pat)
    print(s.getvalue()[:3500])
