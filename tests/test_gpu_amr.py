"""End-to-end AMR parity on the GPU against the reference's golden runs:
identical grids (patch boxes per level), identical raw flag counts and
cell-step accounting; solution bitwise equal with the EXACT step variant and
within 1e-12 norm-relative (BASELINE.json north_star) with the FAST one."""
import numpy as np
import pytest

from tests.amr_cases import CASES
from tests.golden_io import load
from tests.helpers import norm_rel

AMR = load("amr.npz")
pytestmark = pytest.mark.gpu


def build_eq(case):
    from paper_1511_03645_b200 import equations as E
    if case["system"] == "swe":
        return E.SweLinear2D(E.SweMaterialModel(case["material"], sea_level=0.0, gravity=9.81))
    model = E.AcousticsMaterialModel(*case["material"])
    return E.Acoustics1D(model) if case["ndim"] == 1 else E.Acoustics2D(model)


def run(name, variant, adjoint_from_golden=True):
    from paper_1511_03645_b200 import amr
    h, ctx, dt, case = setup(name, variant, adjoint_from_golden)
    out = []
    for step in range(case["steps"]):
        amr.advance_hierarchy(h, 1, dt, ctx)
        snap = {"nlev": h.num_levels(), "flagged": list(ctx.flagged_per_regrid),
                "cell_steps": [ctx.cell_steps.get(lv, 0) for lv in range(1, 5)]}
        for lev in range(1, h.num_levels() + 1):
            ps = h.patches(lev)
            snap[f"L{lev}_boxes"] = np.array([[*p.spec.lo, *p.spec.hi] for p in ps])
            snap[f"L{lev}_q"] = np.concatenate([p.interior().reshape(p.num_components, -1) for p in ps], axis=1)
        out.append(snap)
    return out


def setup(name, variant, adjoint_from_golden=True):
    """The case's initial hierarchy (init regrids + IC), context and dt."""
    from paper_1511_03645_b200 import adjoint, amr, solver
    from paper_1511_03645_b200.geometry import PatchHierarchy, UniformField
    case = CASES[name]
    g = AMR[name]
    eq = build_eq(case)
    bc = solver.BoundarySpec(*case["bc"])
    nd = case["ndim"]
    window = adjoint.TimeWindow(*case["window"])
    if case["strategy"] == "adjoint":
        if adjoint_from_golden:
            origin = (case["xlim"][0],) if nd == 1 else (case["xlim"][0], case["ylim"][0])
            shp = case["adjoint_shape"]
            dx = (case["xlim"][1] - case["xlim"][0]) / shp[0]
            dy = 0.0 if nd == 1 else (case["ylim"][1] - case["ylim"][0]) / shp[1]
            fields = [UniformField(values=v, origin=origin, dx=dx, dy=dy, time=t)
                      for v, t in zip(g["store_fields"], g["store_times"])]
            store = adjoint.AdjointSnapshotStore(times=g["store_times"], fields=fields, window=window,
                                                 wet=g.get("store_wet"))
        else:
            store = adjoint.solve_adjoint(eq, bc, adjoint.FunctionalSpec(*case["functional"]), window,
                                          case["xlim"], case.get("ylim"), case["adjoint_shape"], t0=0.0,
                                          dt_snap=case["snapshot_dt"])
        strategy = adjoint.AdjointFlagging(store, window, case["tol"])
    elif case["strategy"] == "everywhere":
        strategy = amr.EverywhereFlagging()
    else:
        strategy = amr.SurfaceFlagging(case["tol"])
    ctx = amr.AmrContext(equation=eq, boundary=bc, strategy=strategy, limiter="MC",
                         regrid_interval=case["regrid_interval"], buffer_cells=case["buffer"],
                         efficiency=case["efficiency"], max_patch_edge=case["max_patch_edge"], variant=variant)
    h = PatchHierarchy(xlim=case["xlim"], ylim=case.get("ylim"), base_shape=case["base"],
                       ratios=list(case["ratios"]))
    base = amr.make_patch(h, 1, (0,) * nd, tuple(n - 1 for n in case["base"]), ctx, time=0.0)
    h.levels = [[base]]

    def apply_ic(p):
        cs = p.spec.cell_centers()
        if nd == 1:
            p.interior()[...] = case["ic"](cs[0])
        else:
            X, Y = np.meshgrid(cs[0], cs[1], indexing="ij")
            p.interior()[...] = case["ic"](X, Y)
    apply_ic(base)
    for level in range(2, len(case["ratios"]) + 2):
        amr.regrid(h, level, ctx, deepest=level)
        for p in h.patches(level):
            apply_ic(p)
        if not h.patches(level):
            break
    assert ctx.flagged_per_regrid == list(g["init_flagged"])
    dt = solver.select_dt(h, eq, 0.9)
    assert dt == g["dt"]
    return h, ctx, dt, case


def check(name, out, exact):
    g = AMR[name]
    for step, snap in enumerate(out):
        assert snap["nlev"] == g[f"s{step}_nlev"]
        assert snap["flagged"] == list(g[f"s{step}_flagged"]), (step, snap["flagged"])
        assert snap["cell_steps"] == list(g[f"s{step}_cell_steps"])
        for lev in range(1, snap["nlev"] + 1):
            assert np.array_equal(snap[f"L{lev}_boxes"], g[f"s{step}_L{lev}_boxes"]), (step, lev)
            got, want = snap[f"L{lev}_q"], g[f"s{step}_L{lev}_q"]
            if exact:
                assert np.array_equal(got, want), (step, lev, norm_rel(got, want))
            else:
                assert norm_rel(got, want) <= 1e-12, (step, lev, norm_rel(got, want))


@pytest.mark.parametrize("name", sorted(CASES))
def test_amr_exact_variant_bitwise(name):
    from paper_1511_03645_b200 import _lib
    check(name, run(name, _lib.VARIANT_EXACT), exact=True)


@pytest.mark.parametrize("name", sorted(CASES))
def test_amr_fast_variant(name):
    from paper_1511_03645_b200 import _lib
    check(name, run(name, _lib.VARIANT_FAST), exact=False)


@pytest.mark.parametrize("name", [n for n in sorted(CASES) if CASES[n]["strategy"] == "adjoint"])
def test_solve_adjoint_matches_reference_store(name):
    """Device solve_adjoint (reversed f-wave K1 + K2 loop into the HBM ring)."""
    from paper_1511_03645_b200 import adjoint, solver
    case = CASES[name]
    g = AMR[name]
    eq = build_eq(case)
    bc = solver.BoundarySpec(*case["bc"])
    old = solver.DEFAULT_VARIANT
    from paper_1511_03645_b200 import _lib
    try:
        solver.DEFAULT_VARIANT = _lib.VARIANT_EXACT
        st = adjoint.solve_adjoint(eq, bc, adjoint.FunctionalSpec(*case["functional"]),
                                   adjoint.TimeWindow(*case["window"]), case["xlim"], case.get("ylim"),
                                   case["adjoint_shape"], t0=0.0, dt_snap=case["snapshot_dt"])
    finally:
        solver.DEFAULT_VARIANT = old
    assert np.array_equal(st.times, g["store_times"])
    vals = np.stack([f.values for f in st.fields])
    assert np.array_equal(vals, g["store_fields"])
