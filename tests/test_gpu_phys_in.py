"""Physical ghost fill inside the step launch (ADJ_STEP_PHYS_IN, advance_uniform
on a patch spanning its level): each warp job writes the physical ghost cells
its strip reads, as fill_ghost_physical (solver.py:125-146) would, then
marches.  Checked two ways: (1) one launch leaves q_in's ghosts bitwise
equal to a separate K2 physical fill of the same state, and q_out equal to
the fill + step pair, for every side rule; (2) advance_uniform runs
(graph-replayed pairs, odd counts) with and without it agree on the whole
ghost-inclusive patch, forward and adjoint forms.  The step outputs are
compared at the FAST tolerance (1e-12 norm-relative): the launch with the
fill is its own instantiation of the strip kernel, and FMA contraction may
differ between instantiations."""
import numpy as np
import pytest

from tests.helpers import make_equation, norm_rel, patch_from_arrays

pytestmark = pytest.mark.gpu

SIDES = [("outflow", "outflow", "outflow", "outflow"), ("wall", "wall", "wall", "wall"),
         ("wall", "outflow", "outflow", "wall"), ("periodic", "periodic", "wall", "outflow"),
         ("outflow", "wall", "periodic", "periodic"), ("periodic", "periodic", "periodic", "periodic")]


def _patch(name, nx, ny, seed):
    rng = np.random.default_rng(seed)
    swe = name.startswith("swe")
    q = rng.standard_normal((3, nx + 4, ny + 4))
    if swe:
        depth = rng.uniform(50.0, 400.0, (nx + 4, ny + 4))
        aux = np.stack([np.sqrt(9.81 * depth), depth])
    else:
        rho = rng.uniform(0.8, 1.5, (nx + 4, ny + 4))
        bulk = rng.uniform(1.0, 4.0, (nx + 4, ny + 4))
        c = np.sqrt(bulk / rho)
        aux = np.stack([c, rho * c, rho, bulk])
    eq = make_equation(name)
    h, p = patch_from_arrays(q, aux, swe, 1.0 / nx, 1.0 / ny)
    return h, p, eq


def _box(st, t):
    off, NX, NY, pitch = st.boxes[0]
    return t[: st.m * st.plane].view(st.m, -1)[:, off: off + NX * pitch].view(st.m, NX, pitch)[:, :, :NY]


@pytest.mark.parametrize("sides", SIDES)
@pytest.mark.parametrize("name", ["ac2d", "swe_wet", "ac2d_adj_rev"])
@pytest.mark.parametrize("shape", [(37, 70), (130, 33), (3, 5)])
def test_launch_fills_physical_ghosts(name, sides, shape):
    import torch
    from paper_1511_03645_b200 import _lib, device, solver
    nx, ny = shape
    h, p, eq = _patch(name, nx, ny, 3)
    bc = solver.BoundarySpec(*sides)
    st = solver.store_of(p)
    st.sync_in()
    dt = 0.2 * min(p.spec.dx, p.spec.dy) / float(np.max(p.aux.c))
    # reference: separate fill, then the step
    base = st.buf[st.cur].clone()
    device.fill_physical(st, bc, eq, (nx, ny))
    filled = st.buf[st.cur].clone()
    out = st._free(st.cur)
    device.launch_step(st, dt, eq, "MC", _lib.VARIANT_FAST, out, accumulate=True)
    want = st.buf[out].clone()
    # fused: the launch fills q_in's ghosts itself
    st.buf[st.cur].copy_(base)
    st.buf[out].zero_()
    device.launch_step(st, dt, eq, "MC", _lib.VARIANT_FAST, out, accumulate=True, phys_in=(bc, eq, (nx, ny)))
    torch.cuda.synchronize()
    assert torch.equal(_box(st, st.buf[st.cur]), _box(st, filled))
    g = 2
    got_i = _box(st, st.buf[out])[:, g:-g, g:-g].cpu().numpy()
    want_i = _box(st, want)[:, g:-g, g:-g].cpu().numpy()
    assert norm_rel(got_i, want_i) <= 1e-12


@pytest.mark.parametrize("sides", SIDES[:4])
@pytest.mark.parametrize("name", ["swe_wet", "ac2d", "swe_adj_rev"])
def test_advance_uniform_same_with_and_without(name, sides):
    from paper_1511_03645_b200 import _lib, solver
    res = []
    for on in (True, False):
        solver.USE_PHYS_IN = on
        try:
            nx, ny = 64, 96
            h, p, eq = _patch(name, nx, ny, 5)
            bc = solver.BoundarySpec(*sides)
            dt = 0.2 * min(p.spec.dx, p.spec.dy) / float(np.max(p.aux.c))
            for n in (5, 6, 1, 3):
                solver.advance_uniform(p, eq, bc, (nx, ny), dt, n, "MC", _lib.VARIANT_FAST)
            res.append(np.array(p.state))
        finally:
            solver.USE_PHYS_IN = True
    assert norm_rel(res[0], res[1]) <= 1e-12
