"""K1's homogeneous-material instantiation (ADJ_STEP_UNIFORM_MAT): on a level
whose aux planes are constant the strip kernel computes the material terms
once per strip instead of per cell.  Same functions on the same values; FMA
contraction may differ between instantiations, so the step is compared with
the per-cell instantiation at 1e-14 norm-relative and with the oracle
(solver.py:442-512) at the FAST tolerance (1e-12), through the fused
restriction and the in-launch physical fill, and on the homogeneous AMR cases
(whose reference parity tests/test_gpu_amr.py checks with the flag on)."""
import numpy as np
import pytest

from oracle import adjamr_oracle as O
from tests.helpers import make_equation, norm_rel, patch_from_arrays

pytestmark = pytest.mark.gpu


def _patch(nx, ny, seed, c=2.0, z=3.0, dx=None, dy=None, uniform=True):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((3, nx + 4, ny + 4))
    rho, bulk = z / c, z * c
    aux = np.stack([np.full((nx + 4, ny + 4), v) for v in (c, z, rho, bulk)])
    if not uniform:
        aux[1, nx // 2, ny // 3] *= 1.0 + 1e-15 * 4      # one cell off by a few ulps
    eq = make_equation("ac2d")
    h, p = patch_from_arrays(q, aux, False, dx or 1.0 / nx, dy or 1.0 / ny)
    return h, p, eq, q, aux


def _step(p, eq, dt, limiter, on):
    from paper_1511_03645_b200 import _lib, device, solver
    old = device.USE_UNIFORM_MAT
    device.USE_UNIFORM_MAT = on
    try:
        st = solver.store_of(p)
        assert (st.uniform_mat is not None) == on
        solver.step_patch(p, dt, eq, limiter, variant=_lib.VARIANT_FAST)
        return np.array(p.state, copy=True)
    finally:
        device.USE_UNIFORM_MAT = old


@pytest.mark.parametrize("limiter", ["MC", "minmod", "superbee", "none"])
@pytest.mark.parametrize("shape,dxy", [((70, 37), None), ((33, 130), (0.01, 0.013)), ((5, 3), None)])
def test_uniform_step_equals_per_cell_and_oracle(limiter, shape, dxy):
    nx, ny = shape
    dx, dy = dxy if dxy else (None, None)
    outs = []
    for on in (True, False):
        h, p, eq, q, aux = _patch(nx, ny, 5, dx=dx, dy=dy)
        dt = 0.4 * min(p.spec.dx, p.spec.dy) / 2.0
        outs.append(_step(p, eq, dt, limiter, on))
    assert norm_rel(outs[0], outs[1]) <= 1e-14
    want, _ = O.step_2d(q, aux, dt, p.spec.dx, p.spec.dy, O.AC2D, False, False, limiter)
    assert norm_rel(outs[0], want) <= 1e-12


def test_nearly_uniform_material_is_not_uniform():
    from paper_1511_03645_b200 import solver
    h, p, eq, q, aux = _patch(40, 40, 1, uniform=False)
    assert solver.store_of(p).uniform_mat is None
    h, p, eq, q, aux = _patch(40, 40, 1)
    assert solver.store_of(p).uniform_mat == (2.0, 3.0)


@pytest.mark.parametrize("sides", [("wall", "outflow", "outflow", "wall"), ("periodic", "periodic", "wall", "wall")])
def test_advance_uniform_same_with_and_without(sides):
    """advance_uniform (in-launch physical fill, graph replay) on a homogeneous level."""
    from paper_1511_03645_b200 import _lib, device, solver
    outs = []
    for on in (True, False):
        old = device.USE_UNIFORM_MAT
        device.USE_UNIFORM_MAT = on
        try:
            h, p, eq, q, aux = _patch(96, 64, 2)
            bc = solver.BoundarySpec(*sides)
            dt = 0.45 * min(p.spec.dx, p.spec.dy) / 2.0
            solver.advance_uniform(p, eq, bc, (96, 64), dt, 7, "MC", _lib.VARIANT_FAST)
            outs.append(np.array(p.state, copy=True))
        finally:
            device.USE_UNIFORM_MAT = old
    assert norm_rel(outs[0], outs[1]) <= 1e-13


@pytest.mark.parametrize("name", ["ac2d_adjoint", "ac2d_everywhere"])
def test_amr_same_with_and_without(name):
    """Homogeneous AMR cases (packed jobs, fused restriction): identical runs."""
    from paper_1511_03645_b200 import _lib, device
    from tests.test_gpu_amr import run
    res = []
    for on in (True, False):
        old = device.USE_UNIFORM_MAT
        device.USE_UNIFORM_MAT = on
        try:
            res.append(run(name, _lib.VARIANT_FAST))
        finally:
            device.USE_UNIFORM_MAT = old
    for a, b in zip(*res):
        assert a["nlev"] == b["nlev"] and a["flagged"] == b["flagged"]
        for lev in range(1, a["nlev"] + 1):
            assert np.array_equal(a[f"L{lev}_boxes"], b[f"L{lev}_boxes"])
            assert norm_rel(a[f"L{lev}_q"], b[f"L{lev}_q"]) <= 1e-13
