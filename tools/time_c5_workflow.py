"""Inclusive wall time of the host phases of the C5 full workflow (no profiler
overhead): key functions are wrapped with perf_counter timers (the GPU is
synchronised around each wrapped call so device work is charged where it is
launched)."""
import collections, functools, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, adjoint, amr, device, solver

T = collections.defaultdict(float)
N = collections.Counter()


def wrap(mod, name, label=None, sync=True):
    f = getattr(mod, name)
    label = label or f"{mod.__name__.split('.')[-1]}.{name}"

    @functools.wraps(f)
    def g(*a, **k):
        if sync:
            torch.cuda.synchronize()
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            if sync:
                torch.cuda.synchronize()
            T[label] += time.perf_counter() - t
            N[label] += 1
    setattr(mod, name, g)


steps = int(sys.argv[1]) if len(sys.argv) > 1 else 9
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
Tf = steps * dt
window = adjoint.TimeWindow(0.0, Tf)
store = adjoint.solve_adjoint(eq, ctx.boundary, adjoint.FunctionalSpec("box", (0.6, 0.7, 0.3, 0.4), (1.0, 0.0, 0.0)),
                              window, (0.0, 1.0), (0.0, 1.0), (1024, 1024), t0=0.0, dt_snap=Tf / 64,
                              keep_on_device=True)
ctx.strategy = adjoint.AdjointFlagging(store, window, 1e-9, time_interp=True)
ctx.regrid_interval = 4
ctx.max_patch_edge = 64
for mod, name in [(amr, "regrid"), (amr, "make_patches"), (solver, "sample_patches_material"),
                  (amr, "_fill_new_level"), (amr, "_device_level_mask"), (amr, "cluster"),
                  (amr, "_allowed_rectangles"),
                  (amr, "fill_level_ghosts"), (amr, "step_level"), (amr, "_fused_restrict"),
                  (amr, "restrict_fine_to_coarse"), (device, "flag_level_mask"),
                  (adjoint, "flag_level"), (device, "axis_weight_tables"), (device, "_dev_table"),
                  (amr, "build_ghost_rects"), (device, "restrict_cells"), (amr, "_box_overlaps"),
                  (device, "copy_rects"), (device, "coarse_rects"), (solver, "_finish_material"),
                  (device, "flag_axis_tables"), (device, "region_tables"), (amr, "_restrict_rects"),
                  (device, "launch_flag")]:
    wrap(mod, name)
for cls, name in [(device.LevelStore, "__init__"), (device.RectTable, "__init__"),
                  (amr.LevelPlan, "__init__"), (device.GhostPlan, "__init__"),
                  (device.FusedRestrict, "__init__"), (device.RestrictPlan, "__init__"),
                  (amr.Patch, "__init__"),
                  (device.LevelStore, "tiles"), (device.LevelStore, "static_speed"),
                  (device.LevelStore, "edges_table")]:
    f = getattr(cls, name)
    lab = f"{cls.__name__}.{name}"

    def mk(f, lab):
        @functools.wraps(f)
        def g(*a, **k):
            torch.cuda.synchronize()
            t = time.perf_counter()
            try:
                return f(*a, **k)
            finally:
                torch.cuda.synchronize()
                T[lab] += time.perf_counter() - t
                N[lab] += 1
        return g
    setattr(cls, name, mk(f, lab))
torch.cuda.synchronize()
times = []
for step in range(steps):
    if step == 1:
        T.clear(); N.clear()
    t0 = time.perf_counter()
    nreg = len(ctx.flagged_per_regrid)
    amr.advance_hierarchy(h, 1, dt, ctx)
    torch.cuda.synchronize()
    times.append((round(1e3 * (time.perf_counter() - t0), 2), len(ctx.flagged_per_regrid) > nreg))
print("step ms (regrid?)", times)
print("patches", [len(h.patches(l)) for l in (1, 2, 3)])
for k in sorted(T, key=lambda k: -T[k]):
    print(f"{k:40s} n={N[k]:5d} total={1e3 * T[k]:9.2f} ms  per={1e3 * T[k] / N[k]:8.3f} ms")
