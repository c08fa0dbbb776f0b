import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, adjoint, amr
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
T = 9 * dt
window = adjoint.TimeWindow(0.0, T)
store = adjoint.solve_adjoint(eq, ctx.boundary, adjoint.FunctionalSpec("box", (0.6, 0.7, 0.3, 0.4), (1.0, 0.0, 0.0)),
                              window, (0.0, 1.0), (0.0, 1.0), (1024, 1024), t0=0.0, dt_snap=T / 64, keep_on_device=True)
ctx.strategy = adjoint.AdjointFlagging(store, window, 1e-9, time_interp=True)
ctx.max_patch_edge = 64
amr.advance_hierarchy(h, 1, dt, ctx)
torch.cuda.synchronize()
for rep in range(2):
    pr = cProfile.Profile()
    t = time.perf_counter()
    pr.enable()
    amr.regrid(h, 2, ctx)
    torch.cuda.synchronize()
    pr.disable()
    print("regrid s", time.perf_counter() - t, [len(h.patches(l)) for l in (1, 2, 3)])
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(28)
    print(s.getvalue()[:6000])
