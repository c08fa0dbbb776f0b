"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (needs /root/reference, never on the GPU box):
    python tests/golden/make_golden.py
Writes tests/golden/*.npz (committed).  Each fixture stores the seeded
inputs in the device layout (q planes incl. ghosts, aux planes) and the
reference's outputs, so the oracle and the CUDA kernels can be checked
against the reference itself without importing it.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from adjamr import adjoint as radj          # noqa: E402
from adjamr import amr as ramr              # noqa: E402
from adjamr import equations as req         # noqa: E402
from adjamr import geometry as rgeo         # noqa: E402
from adjamr import solver as rsol           # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def aux_planes(aux):
    if hasattr(aux, "wet"):
        return np.stack([aux.c, aux.depth])
    return np.stack([aux.c, aux.z, aux.rho, aux.bulk])


def ac_model(kind):
    if kind == "hetero":
        return req.AcousticsMaterialModel(
            lambda x, y=None: 1.0 + 3.0 * (np.asarray(x) > 0.3) + 0.5 * np.sin(3.0 * np.asarray(x) + (0 if y is None else 2.0 * np.asarray(y))) ** 2,
            lambda x, y=None: np.where(np.asarray(x) + (0 if y is None else np.asarray(y)) < 0.7, 1.0, 1.5)
            + 0.2 * np.cos(2.0 * np.asarray(x)))
    return req.AcousticsMaterialModel(lambda x, y=None: np.full_like(np.asarray(x, float), 4.0),
                                      lambda x, y=None: np.ones_like(np.asarray(x, float)))


def swe_model(dry):
    def bathy(x, y):
        x = np.asarray(x, float)
        y = np.asarray(y, float)
        b = -50.0 - 30.0 * np.sin(2.0 * x) * np.cos(3.0 * y)
        if dry:
            b = np.where((x - 0.8) ** 2 + (y - 0.3) ** 2 < 0.06, 5.0, b)
        return b
    return req.SweMaterialModel(bathy, sea_level=0.0, gravity=9.81)


def make_eq(name):
    table = {
        "ac2d": lambda: req.Acoustics2D(ac_model("hetero")),
        "ac2d_adj_rev": lambda: req.Acoustics2D(ac_model("hetero")).adjoint().reversed(),
        "ac2d_adj": lambda: req.Acoustics2D(ac_model("hetero")).adjoint(),
        "ac2d_rev": lambda: req.TimeReversed(req.Acoustics2D(ac_model("hetero"))),
        "swe_wet": lambda: req.SweLinear2D(swe_model(False)),
        "swe_dry": lambda: req.SweLinear2D(swe_model(True)),
        "swe_adj_rev": lambda: req.SweLinear2D(swe_model(True)).adjoint().reversed(),
        "swe_wet_adj_rev": lambda: req.SweLinear2D(swe_model(False)).adjoint().reversed(),
        "ac1d": lambda: req.Acoustics1D(ac_model("hetero")),
        "ac1d_adj_rev": lambda: req.Acoustics1D(ac_model("hetero")).adjoint().reversed(),
    }
    return table[name]()


def make_patch(eq, shape, bc, lo=None, level_shape=None, xlim=(0.0, 1.2), ylim=(0.0, 1.0)):
    nd = len(shape)
    h = rgeo.PatchHierarchy(xlim=xlim, ylim=None if nd == 1 else ylim,
                            base_shape=tuple(level_shape or shape), ratios=[])
    lo = lo or (0,) * nd
    spec = h.make_spec(1, lo, tuple(l + n - 1 for l, n in zip(lo, shape)))
    p = rgeo.Patch(spec, eq.m)
    rsol.sample_patch_material(p, eq, bc, tuple(level_shape or shape))
    return h, p


def rand_state(rng, p, scale=1.0):
    q = p.interior()
    xs = p.spec.cell_centers()
    if p.spec.ndim == 2:
        X, Y = np.meshgrid(xs[0], xs[1], indexing="ij")
        base = np.exp(-30 * ((X - 0.5) ** 2 + (Y - 0.5) ** 2))
    else:
        base = np.exp(-30 * (xs[0] - 0.5) ** 2)
    for c in range(q.shape[0]):
        q[c] = scale * (base * (1 + c) * 0.5 + 0.3 * rng.normal(size=base.shape))


def step_cases(rng):
    out = {}
    cases = [
        ("ac2d", "MC", (22, 19), rsol.BoundarySpec("wall", "outflow", "outflow", "wall")),
        ("ac2d", "minmod", (17, 23), rsol.BoundarySpec()),
        ("ac2d", "superbee", (20, 20), rsol.BoundarySpec("outflow", "outflow", "outflow", "outflow")),
        ("ac2d", "none", (16, 21), rsol.BoundarySpec()),
        ("ac2d_adj_rev", "MC", (21, 18), rsol.BoundarySpec("wall", "outflow", "wall", "outflow")),
        ("ac2d_adj", "MC", (18, 18), rsol.BoundarySpec()),
        ("ac2d_rev", "superbee", (19, 17), rsol.BoundarySpec()),
        ("swe_wet", "MC", (24, 20), rsol.BoundarySpec("outflow", "outflow", "wall", "wall")),
        ("swe_dry", "MC", (26, 22), rsol.BoundarySpec()),
        ("swe_dry", "minmod", (20, 25), rsol.BoundarySpec("outflow", "wall", "outflow", "wall")),
        ("swe_adj_rev", "MC", (23, 21), rsol.BoundarySpec()),
        ("swe_wet_adj_rev", "superbee", (21, 21), rsol.BoundarySpec("outflow", "outflow", "outflow", "outflow")),
        ("ac1d", "MC", (64,), rsol.BoundarySpec("outflow", "wall")),
        ("ac1d", "none", (40,), rsol.BoundarySpec()),
        ("ac1d_adj_rev", "MC", (57,), rsol.BoundarySpec("wall", "outflow")),
        ("ac1d_adj_rev", "superbee", (33,), rsol.BoundarySpec()),
    ]
    for k, (eqn, lim, shape, bc) in enumerate(cases):
        eq = make_eq(eqn)
        h, p = make_patch(eq, shape, bc, xlim=(0.0, 1.2) if eqn.startswith("ac") else (0.0, 1.2))
        rand_state(rng, p, scale=1.0 if eqn.startswith("ac") else 0.3)
        rsol.fill_ghost_physical(p, bc, eq, shape)
        q_in = p.state.copy()
        cmax = float(np.max(p.aux.c))
        dt = 0.8 * min(p.spec.widths) / cmax
        res = rsol.step_patch(p, dt, eq, lim)
        key = f"step{k:02d}"
        out[key] = dict(name=eqn, limiter=lim, q_in=q_in, aux=aux_planes(p.aux), dt=dt,
                        dx=p.spec.dx, dy=p.spec.dy, q_out=p.state.copy(), cfl=res.max_courant,
                        gravity=getattr(p.aux, "gravity", 0.0), bc=np.array([bc.left, bc.right, bc.bottom, bc.top]))
    return out


def integrate_cases(rng):
    out = {}
    for k, (eqn, shape, bc, T) in enumerate([
            ("ac2d", (30, 26), rsol.BoundarySpec("wall", "outflow", "wall", "outflow"), 0.25),
            ("swe_dry", (28, 28), rsol.BoundarySpec(), 0.01),
            ("ac1d", (80,), rsol.BoundarySpec("outflow", "outflow"), 0.3)]):
        eq = make_eq(eqn)
        h, p = make_patch(eq, shape, bc)
        rand_state(rng, p, scale=1.0 if eqn.startswith("ac") else 0.3)
        q0 = p.state.copy()
        steps = []
        rsol.integrate_patch(p, eq, bc, shape, T, limiter="MC", on_step=lambda pp: steps.append(pp.time))
        out[f"integ{k}"] = dict(name=eqn, q0=q0, aux=aux_planes(p.aux), t_end=T, bc=np.array([bc.left, bc.right, bc.bottom, bc.top]),
                                q_out=p.state.copy(), nsteps=len(steps), dx=p.spec.dx, dy=p.spec.dy,
                                gravity=getattr(p.aux, "gravity", 0.0))
    return out


def ghost_cases(rng):
    out = {}
    # physical fills on patches touching various edges
    eq = make_eq("ac2d")
    for k, (lo, shape, level_shape, bc) in enumerate([
            ((0, 0), (10, 12), (10, 12), rsol.BoundarySpec("wall", "outflow", "outflow", "wall")),
            ((0, 5), (8, 7), (20, 12), rsol.BoundarySpec("wall", "wall", "wall", "wall")),
            ((12, 0), (8, 6), (20, 12), rsol.BoundarySpec("outflow", "outflow", "wall", "outflow"))]):
        h, p = make_patch(eq, shape, bc, lo=lo, level_shape=level_shape)
        p.state[...] = rng.normal(size=p.state.shape)
        q_in = p.state.copy()
        rsol.fill_ghost_physical(p, bc, eq, level_shape)
        out[f"phys{k}"] = dict(q_in=q_in, q_out=p.state.copy(), lo=np.array(lo), shape=np.array(shape),
                               level_shape=np.array(level_shape), bc=np.array([bc.left, bc.right, bc.bottom, bc.top]))
    # coarse -> fine space-time interpolation (solver.py:227-286)
    h = rgeo.PatchHierarchy(xlim=(0.0, 2.0), ylim=(0.0, 1.5), base_shape=(16, 12), ratios=[2])
    bc = rsol.BoundarySpec()
    cps = []
    for lo, hi in [((0, 0), (7, 11)), ((8, 0), (15, 11))]:
        cp = rgeo.Patch(h.make_spec(1, lo, hi), 3)
        rsol.sample_patch_material(cp, eq, bc, (16, 12))
        cp.state[...] = rng.normal(size=cp.state.shape)
        cp.save_old()
        cp.time = 0.4
        cp.state[...] = rng.normal(size=cp.state.shape)
        cps.append(cp)
    fp = rgeo.Patch(h.make_spec(2, (10, 6), (21, 17)), 3)
    rsol.sample_patch_material(fp, eq, bc, (32, 24))
    h.levels = [cps, [fp]]
    res = {}
    for t in (0.0, 0.13, 0.4):
        fp.state[...] = 0.0
        rsol.fill_ghost_from_coarse(fp, h, t)
        res[f"t{t}"] = fp.state.copy()
    out["coarse0"] = dict(c0_old=cps[0].state_old, c0_new=cps[0].state, c1_old=cps[1].state_old, c1_new=cps[1].state,
                          t_list=np.array([0.0, 0.13, 0.4]), f_t0=res["t0.0"], f_t1=res["t0.13"], f_t2=res["t0.4"])
    return out


def restrict_cases(rng):
    out = {}
    for k, (eqn, r) in enumerate([("ac2d", 2), ("ac2d", 4), ("swe_dry", 2), ("swe_dry", 4),
                                  ("ac2d", 4), ("swe_dry", 4), ("ac2d", 2)]):
        eq = make_eq(eqn)
        bc = rsol.BoundarySpec()
        h = rgeo.PatchHierarchy(xlim=(0.0, 1.2), ylim=(0.0, 1.0), base_shape=(12, 10), ratios=[r])
        cp = rgeo.Patch(h.make_spec(1, (0, 0), (11, 9)), 3)
        rsol.sample_patch_material(cp, eq, bc, (12, 10))
        cp.state[...] = rng.normal(size=cp.state.shape)
        fps = []
        boxes = [((2 * r, 1 * r), (6 * r - 1, 5 * r - 1)), ((7 * r, 3 * r), (11 * r - 1, 9 * r - 1))]
        if k >= 4:   # coarse overlaps one cell wide in y / x (numpy reduces them differently)
            boxes = [((2 * r, 1 * r), (6 * r - 1, 2 * r - 1)), ((7 * r, 3 * r), (8 * r - 1, 9 * r - 1))]
        for lo, hi in boxes:
            fp = rgeo.Patch(h.make_spec(2, lo, hi), 3)
            rsol.sample_patch_material(fp, eq, bc, (12 * r, 10 * r))
            fp.state[...] = rng.normal(size=fp.state.shape)
            fps.append(fp)
        h.levels = [[cp], fps]
        before = cp.state.copy()
        ramr.restrict_fine_to_coarse(h, 1)
        out[f"restrict{k}"] = dict(name=eqn, ratio=r, c_in=before, c_out=cp.state.copy(), c_aux=aux_planes(cp.aux),
                                   f0=fps[0].state.copy(), f1=fps[1].state.copy(), f0_aux=aux_planes(fps[0].aux),
                                   f1_aux=aux_planes(fps[1].aux),
                                   f_lohi=np.array([[*fps[0].spec.lo, *fps[0].spec.hi], [*fps[1].spec.lo, *fps[1].spec.hi]]))
    return out


def flag_cases(rng):
    out = {}
    # 2D acoustics, adjoint grid coarser than the forward patch
    for k, (eqn, nxa, nya, shape, lo, dry_adj) in enumerate([
            ("ac2d", 24, 20, (30, 26), (0, 0), False),
            ("ac2d", 50, 40, (17, 13), (21, 9), False),
            ("swe_dry", 30, 30, (26, 22), (0, 0), True)]):
        eq = make_eq(eqn)
        bc = rsol.BoundarySpec()
        level_shape = (48, 40)
        h, p = make_patch(eq, shape, bc, lo=lo, level_shape=level_shape)
        p.state[...] = rng.normal(size=p.state.shape)
        times = np.linspace(0.0, 2.0, 9)
        fields = [rgeo.UniformField(values=rng.normal(size=(3, nxa, nya)), origin=(0.0, 0.0),
                                    dx=1.2 / nxa, dy=1.0 / nya, time=t) for t in times]
        wet = None
        if dry_adj:
            wet = rng.random((nxa, nya)) > 0.2
        store = radj.AdjointSnapshotStore(times=times, fields=fields, window=radj.TimeWindow(1.0, 2.0), wet=wet)
        res = {}
        for t in (0.0, 0.37, 1.5, 2.0):
            idx = radj.query_window_times(t, store.window, store)
            best = radj.inner_product_field(p, t, store, store.window)
            flags = radj.inner_product_flags(p, t, store, store.window, 0.8).flags
            res[t] = (np.array(idx, dtype=np.int64), best, flags)
        d = dict(name=eqn, q=p.state.copy(), aux=aux_planes(p.aux), lo=np.array(lo), shape=np.array(shape),
                 dx=p.spec.dx, dy=p.spec.dy, fields=np.stack([f.values for f in fields]), times=times,
                 a_dx=fields[0].dx, a_dy=fields[0].dy, tol=0.8, t_list=np.array(sorted(res)),
                 adj_wet=wet if wet is not None else np.zeros(0, bool))
        for n, t in enumerate(sorted(res)):
            d[f"idx{n}"], d[f"best{n}"], d[f"flags{n}"] = res[t]
        # time-interpolated values (interpolate_time + inner product arithmetic)
        tint = []
        for t in (0.37, 1.1):
            f = store.interpolate_time(t)
            x = np.broadcast_to(p.spec.cell_centers()[0][:, None], p.spec.shape)
            y = np.broadcast_to(p.spec.cell_centers()[1][None, :], p.spec.shape)
            qh = rgeo.interpolate_uniform(f, x, y)
            tint.append(np.abs(np.sum(qh * p.interior(), axis=0)))
        d["interp_t"] = np.array([0.37, 1.1])
        d["interp_val"] = np.stack(tint)
        out[f"flag{k}"] = d
    # 1D
    eq = make_eq("ac1d")
    h, p = make_patch(eq, (50,), rsol.BoundarySpec(), lo=(10,), level_shape=(80,), xlim=(0.0, 2.0))
    p.state[...] = rng.normal(size=p.state.shape)
    times = np.linspace(0.0, 1.0, 6)
    fields = [rgeo.UniformField(values=rng.normal(size=(2, 37)), origin=(0.0,), dx=2.0 / 37, dy=0.0, time=t)
              for t in times]
    store = radj.AdjointSnapshotStore(times=times, fields=fields, window=radj.TimeWindow(0.5, 1.0))
    idx = radj.query_window_times(0.3, store.window, store)
    best = radj.inner_product_field(p, 0.3, store, store.window)
    out["flag1d"] = dict(q=p.state.copy(), lo=np.array([10]), shape=np.array([50]), dx=p.spec.dx,
                         fields=np.stack([f.values for f in fields]), times=times, a_dx=2.0 / 37,
                         idx=np.array(idx), best=best)
    # window query known answers on random grids
    qs = []
    for _ in range(300):
        n = int(rng.integers(2, 30))
        t0 = float(rng.uniform(-1, 1))
        dts = float(rng.uniform(0.01, 0.5))
        times = t0 + dts * np.arange(n)
        tf = float(times[-1])
        ts = float(rng.uniform(times[0], tf))
        t = float(rng.uniform(times[0] - 0.3, tf + 0.3)) if rng.random() < 0.7 else float(times[int(rng.integers(0, n))])
        fields = [rgeo.UniformField(values=np.zeros((1, 1)), origin=(0.0,), dx=1.0, dy=0.0, time=tt) for tt in times]
        st = radj.AdjointSnapshotStore(times=times, fields=fields, window=radj.TimeWindow(ts, tf))
        idx = radj.query_window_times(t, st.window, st)
        qs.append((t, ts, tf, times, idx))
    out["window"] = dict(
        t=np.array([q[0] for q in qs]), ts=np.array([q[1] for q in qs]), tf=np.array([q[2] for q in qs]),
        times=np.array([np.pad(q[3], (0, 30 - len(q[3])), constant_values=np.nan) for q in qs]),
        ntimes=np.array([len(q[3]) for q in qs]),
        idx=np.array([np.pad(np.array(q[4], dtype=np.int64), (0, 32 - len(q[4])), constant_values=-1) for q in qs]))
    return out


def save(name, cases):
    flat = {}
    for key, d in cases.items():
        for f, v in d.items():
            flat[f"{key}.{f}"] = np.asarray(v)
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **flat)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB, {len(cases)} cases)")


def main():
    rng = np.random.default_rng(20240601)
    save("step.npz", step_cases(rng))
    save("integrate.npz", integrate_cases(rng))
    save("ghost.npz", ghost_cases(rng))
    save("restrict.npz", restrict_cases(rng))
    save("flag.npz", flag_cases(rng))


if __name__ == "__main__":
    main()
