import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, adjoint, amr, device
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
steps = 13
T = steps * dt
window = adjoint.TimeWindow(0.0, T)
store = adjoint.solve_adjoint(eq, ctx.boundary, adjoint.FunctionalSpec("box", (0.6, 0.7, 0.3, 0.4), (1.0, 0.0, 0.0)),
                              window, (0.0, 1.0), (0.0, 1.0), (1024, 1024), t0=0.0, dt_snap=T / 64, keep_on_device=True)
ctx.strategy = adjoint.AdjointFlagging(store, window, 1e-9, time_interp=True)
ctx.regrid_interval = 4
ctx.max_patch_edge = 64
for k in range(steps - 1):
    t0 = time.perf_counter()
    amr.advance_hierarchy(h, 1, dt, ctx)
    torch.cuda.synchronize()
    gc.collect()
    live = sum(1 for o in gc.get_objects() if isinstance(o, device.LevelStore))
    print(k, round(1e3 * (time.perf_counter() - t0), 1), "ms live stores", live,
          "alloc MB", torch.cuda.memory_allocated() >> 20, "reserved MB", torch.cuda.memory_reserved() >> 20)
