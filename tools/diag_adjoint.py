"""Diagnostic: product integrate loop (exact variant) vs the CPU oracle, step by step."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import adjamr_oracle as O  # noqa: E402
from paper_1511_03645_b200 import _lib, adjoint, solver  # noqa: E402
from paper_1511_03645_b200.geometry import Patch, PatchHierarchy  # noqa: E402
from tests.amr_cases import CASES  # noqa: E402
from tests.test_gpu_amr import build_eq  # noqa: E402

for name in ("ac1d_adjoint", "ac2d_adjoint"):
    case = CASES[name]
    eq = build_eq(case)
    rev = eq.adjoint().reversed()
    bc = solver.BoundarySpec(*case["bc"])
    nd = case["ndim"]
    shp = case["adjoint_shape"]
    h = PatchHierarchy(xlim=case["xlim"], ylim=case.get("ylim"), base_shape=shp, ratios=[])
    p = Patch(h.make_spec(1, (0,) * nd, tuple(n - 1 for n in shp)), eq.m)
    solver.sample_patch_material(p, rev, bc, shp)
    rng = np.random.default_rng(0)
    p.interior()[...] = rng.normal(size=p.interior().shape)
    q = p.state.copy()
    aux = np.stack(p.aux.planes())
    dt = 0.9 * p.spec.dx / float(np.max(p.aux.c)) * 0.5
    edges = {"xlo": True, "xhi": True, "ylo": True, "yhi": True}
    bcd = dict(zip(("xlo", "xhi", "ylo", "yhi"), (bc.left, bc.right, bc.bottom, bc.top)))
    sysname = O.AC1D if nd == 1 else O.AC2D
    for step in range(6):
        solver.fill_ghost_physical(p, bc, rev, shp)
        q = O.fill_physical(q, 2, edges, bcd, (1,) if nd == 1 else (1, 2))
        st_after_fill = p.state.copy()
        print(name, step, "fill equal", np.array_equal(st_after_fill, q), np.max(np.abs(st_after_fill - q)))
        solver.step_patch(p, dt, rev, "MC", variant=_lib.VARIANT_EXACT)
        if nd == 1:
            q, _ = O.step_1d(q, aux, dt, p.spec.dx, sysname, True, True, "MC")
        else:
            q, _ = O.step_2d(q, aux, dt, p.spec.dx, p.spec.dy, sysname, True, True, "MC")
        got = p.state
        eq_ = np.array_equal(got, q)
        print(name, step, "step equal", eq_, np.max(np.abs(got - q)))
        if not eq_:
            idx = np.argwhere(got != q)[:5]
            print("  first diffs", idx.tolist())
            break
