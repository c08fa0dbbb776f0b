import os, sys, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, adjoint, amr, device, solver
acc = collections.defaultdict(float)
cnt = collections.Counter()
def wrap(mod, name, label=None):
    f = getattr(mod, name)
    label = label or name
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); acc[label] += time.perf_counter() - t0; cnt[label] += 1
        return r
    setattr(mod, name, g)
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
for mod, name in [(amr, "regrid"), (amr, "_device_level_mask"), (amr, "cluster"), (amr, "_allowed_rectangles"),
                  (amr, "make_patch"), (amr, "_fill_new_level"), (amr.LevelPlan, "__init__"),
                  (device.GhostPlan, "__init__"), (device.RestrictPlan, "__init__"), (amr, "fill_level_ghosts"),
                  (amr, "step_level"), (amr, "restrict_fine_to_coarse"), (device.LevelStore, "tiles"),
                  (device.LevelStore, "__init__"), (device.LevelStore, "static_speed"), (amr, "allowed_region_mask")]:
    wrap(mod, name, f"{getattr(mod, '__name__', mod)}.{name}")
t0 = time.perf_counter()
for k in range(steps - 2):
    amr.advance_hierarchy(h, 1, dt, ctx)
torch.cuda.synchronize()
print("total ms", round(1e3 * (time.perf_counter() - t0), 1))
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"{k:28s} {1e3 * v:8.1f} ms  n={cnt[k]}")
