"""Golden end-to-end AMR runs produced by the REFERENCE (build container only).

    python tests/golden/make_golden_amr.py   -> tests/golden/amr.npz

Each case: an adjoint solve (reference solve_adjoint) and a forward AMR run
(base patch + initial regrids as driver.init_hierarchy does, then coarse
steps of advance_hierarchy with select_dt).  Stored: the adjoint store, the
grid (lo, hi per patch per level), interior states, cell_steps and
flagged_per_regrid after every coarse step.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from adjamr import adjoint as radj      # noqa: E402
from adjamr import amr as ramr          # noqa: E402
from adjamr import equations as req     # noqa: E402
from adjamr import geometry as rgeo     # noqa: E402
from adjamr import solver as rsol       # noqa: E402

from tests.amr_cases import CASES       # noqa: E402  (shared case definitions)

OUT = os.path.dirname(os.path.abspath(__file__))


def build_eq(case):
    mats = case["material"]
    if case["system"] == "swe":
        return req.SweLinear2D(req.SweMaterialModel(mats, sea_level=0.0, gravity=9.81))
    model = req.AcousticsMaterialModel(*mats)
    return req.Acoustics1D(model) if case["ndim"] == 1 else req.Acoustics2D(model)


def run_case(name, case):
    eq = build_eq(case)
    bc = rsol.BoundarySpec(*case["bc"])
    nd = case["ndim"]
    window = radj.TimeWindow(*case["window"])
    store = None
    if case["strategy"] == "adjoint":
        store = radj.solve_adjoint(eq, bc, radj.FunctionalSpec(*case["functional"]), window, case["xlim"],
                                   case.get("ylim"), case["adjoint_shape"], t0=0.0,
                                   dt_snap=case["snapshot_dt"], courant_target=0.9, limiter="MC")
        strategy = radj.AdjointFlagging(store, window, case["tol"])
    elif case["strategy"] == "everywhere":
        strategy = ramr.EverywhereFlagging()
    else:
        strategy = ramr.SurfaceFlagging(case["tol"])
    ctx = ramr.AmrContext(equation=eq, boundary=bc, strategy=strategy, limiter="MC",
                          regrid_interval=case["regrid_interval"], buffer_cells=case["buffer"],
                          efficiency=case["efficiency"], max_patch_edge=case["max_patch_edge"])
    h = rgeo.PatchHierarchy(xlim=case["xlim"], ylim=case.get("ylim"), base_shape=case["base"],
                            ratios=list(case["ratios"]))
    base = ramr.make_patch(h, 1, (0,) * nd, tuple(n - 1 for n in case["base"]), ctx, time=0.0)
    h.levels = [[base]]
    ic = case["ic"]

    def apply_ic(p):
        cs = p.spec.cell_centers()
        if nd == 1:
            p.interior()[...] = ic(cs[0])
        else:
            X, Y = np.meshgrid(cs[0], cs[1], indexing="ij")
            p.interior()[...] = ic(X, Y)
    apply_ic(base)
    for level in range(2, len(case["ratios"]) + 2):
        ramr.regrid(h, level, ctx, deepest=level)
        for p in h.patches(level):
            apply_ic(p)
        if not h.patches(level):
            break
    out = {}
    if store is not None:
        out["store_times"] = store.times
        out["store_fields"] = np.stack([f.values for f in store.fields])
        if store.wet is not None:
            out["store_wet"] = store.wet
    out["init_flagged"] = np.array(ctx.flagged_per_regrid, dtype=np.int64)
    dt = rsol.select_dt(h, eq, 0.9)
    out["dt"] = dt
    for step in range(case["steps"]):
        ramr.advance_hierarchy(h, 1, dt, ctx)
        for lev in range(1, h.num_levels() + 1):
            ps = h.patches(lev)
            out[f"s{step}_L{lev}_boxes"] = np.array([[*p.spec.lo, *p.spec.hi] for p in ps], dtype=np.int64)
            out[f"s{step}_L{lev}_q"] = np.concatenate([p.interior().reshape(p.num_components, -1) for p in ps], axis=1)
        out[f"s{step}_nlev"] = h.num_levels()
        out[f"s{step}_flagged"] = np.array(ctx.flagged_per_regrid, dtype=np.int64)
        out[f"s{step}_cell_steps"] = np.array([ctx.cell_steps.get(lv, 0) for lv in range(1, 5)], dtype=np.int64)
    return out


def main():
    flat = {}
    for name, case in CASES.items():
        res = run_case(name, case)
        for k, v in res.items():
            flat[f"{name}.{k}"] = np.asarray(v)
        print(name, "levels", res[f"s{case['steps'] - 1}_nlev"], "flagged", res[f"s{case['steps'] - 1}_flagged"][-4:])
    path = os.path.join(OUT, "amr.npz")
    np.savez_compressed(path, **flat)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
