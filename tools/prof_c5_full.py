"""cProfile of the full C5 workflow (adjoint solve excluded): advance with regrids."""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, adjoint, amr
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = steps * dt
window = adjoint.TimeWindow(0.0, T)
store = adjoint.solve_adjoint(eq, ctx.boundary, adjoint.FunctionalSpec("box", (0.6, 0.7, 0.3, 0.4), (1.0, 0.0, 0.0)),
                              window, (0.0, 1.0), (0.0, 1.0), (1024, 1024), t0=0.0, dt_snap=T / 64, keep_on_device=True)
ctx.strategy = adjoint.AdjointFlagging(store, window, 1e-9, time_interp=True)
ctx.regrid_interval = 4
ctx.max_patch_edge = 64
amr.advance_hierarchy(h, 1, dt, ctx)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for k in range(steps - 1):
    s0 = time.perf_counter()
    amr.advance_hierarchy(h, 1, dt, ctx)
    torch.cuda.synchronize()
    print("step", k, round(1e3 * (time.perf_counter() - s0), 1), "ms", [len(h.patches(l)) for l in (1, 2, 3)])
pr.disable()
print("total s", time.perf_counter() - t0)
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(45)
print(s.getvalue()[:9000])
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000])
