"""FAST K1 on shallow water with dry cells (ADJ_STEP_WET_DRY): the strip
kernel's wet/dry instantiation against the CPU oracle (a restatement of
step_patch_2d with _swe_effective_states / _swe_transverse_material /
dq *= wet, solver.py:357-387, 442-512) and against the EXACT kernel, on
coastlines, islands, isolated dry cells, one-cell wet channels and both-dry
faces.  Tolerance: BASELINE north_star's 1e-12 (norm-relative per component)."""
import numpy as np
import pytest

from oracle import adjamr_oracle as O
from tests.helpers import make_equation, norm_rel, patch_from_arrays

pytestmark = pytest.mark.gpu
G = 9.81


def dry_case(seed, nx=70, ny=45, frac=0.3):
    """Ghost-inclusive (3, nx+4, ny+4) state and (c, depth) planes: a coast
    (dry for x > 0.8 nx), an island, random isolated dry cells and a one-cell
    wet channel through dry land."""
    rng = np.random.default_rng(seed)
    NX, NY = nx + 4, ny + 4
    depth = rng.uniform(50.0, 4000.0, (NX, NY))
    ii, jj = np.meshgrid(np.arange(NX), np.arange(NY), indexing="ij")
    dry = ii > int(0.8 * NX)
    dry |= (ii - NX * 0.4) ** 2 + (jj - NY * 0.5) ** 2 < (0.12 * NY) ** 2
    dry |= rng.random((NX, NY)) < frac * 0.2
    dry[:, NY // 3] |= ii[:, 0] > NX // 2          # a dry wall with
    dry[int(0.6 * NX), NY // 3] = False            # a one-cell gap
    depth = np.where(dry, -rng.uniform(0.0, 50.0, (NX, NY)), depth)
    depth[3, 3] = 0.0                              # depth exactly zero is dry
    c = np.sqrt(G * np.maximum(depth, 0.0))
    q = np.zeros((3, NX, NY))
    q[0] = rng.normal(0.0, 1.0, (NX, NY))
    q[1] = rng.normal(0.0, 50.0, (NX, NY))
    q[2] = rng.normal(0.0, 50.0, (NX, NY))
    return q, np.stack([c, depth])


@pytest.mark.parametrize("limiter", ["MC", "minmod", "superbee", "none"])
@pytest.mark.parametrize("square", [True, False])
@pytest.mark.parametrize("seed", [0, 1])
def test_fast_wet_dry_vs_oracle(limiter, square, seed):
    from paper_1511_03645_b200 import _lib, device, solver
    q, aux = dry_case(seed)
    dx, dy = (1000.0, 1000.0) if square else (1000.0, 750.0)
    dt = 0.45 * min(dx, dy) / float(np.max(aux[0]))
    eq = make_equation("swe_dry", gravity=G)
    _, p = patch_from_arrays(q, aux, True, dx, dy, gravity=G)
    assert solver.store_of(p).any_dry() and device.fast_dry_ok(solver.store_of(p), eq)
    res = solver.step_patch(p, dt, eq, limiter, variant=_lib.VARIANT_FAST)
    want, cfl = O.step_2d(q, aux, dt, dx, dy, O.SWE2D, False, False, limiter, G)
    got = p.state
    assert norm_rel(got, want) <= 1e-12, norm_rel(got, want)
    assert abs(res.max_courant - cfl) <= 1e-14 * max(cfl, 1.0)
    wet = aux[1] > 0
    inner = np.zeros(wet.shape, bool)
    inner[2:-2, 2:-2] = True
    # dry cells keep their state (dq *= wet), ghosts are untouched
    assert np.array_equal(np.abs(got[:, ~wet | ~inner]), np.abs(q[:, ~wet | ~inner]))


def test_fast_wet_dry_multistep_vs_exact():
    """advance_uniform (the step launch fills its input's wall ghosts) over 12
    steps with a coastline: FAST within 1e-12 of EXACT."""
    from paper_1511_03645_b200 import _lib, solver
    outs = []
    for var in (_lib.VARIANT_EXACT, _lib.VARIANT_FAST):
        q, aux = dry_case(5, 200, 160)
        dx = dy = 500.0
        dt = 0.8 * dx / float(np.max(aux[0]))
        eq = make_equation("swe_dry", gravity=G)
        _, p = patch_from_arrays(q, aux, True, dx, dy, gravity=G)
        bc = solver.BoundarySpec("wall", "outflow", "wall", "wall")
        solver.advance_uniform(p, eq, bc, (200, 160), dt, 12, "MC", var)
        outs.append(p.interior().copy())
    assert norm_rel(outs[1], outs[0]) <= 1e-12, norm_rel(outs[1], outs[0])


@pytest.mark.parametrize("limiter", ["MC", "minmod"])
@pytest.mark.parametrize("square", [True, False])
@pytest.mark.parametrize("seed", [0, 3])
def test_fast_wet_dry_adjoint_vs_oracle(limiter, square, seed):
    """The time-reversed f-wave adjoint (solve_adjoint's step) on a level with
    dry cells: the strip kernel's wet/dry instantiation against the oracle."""
    from paper_1511_03645_b200 import _lib, device, solver
    q, aux = dry_case(seed)
    dx, dy = (1000.0, 1000.0) if square else (1000.0, 750.0)
    dt = 0.45 * min(dx, dy) / float(np.max(aux[0]))
    eq = make_equation("swe_adj_rev", gravity=G)
    _, p = patch_from_arrays(q, aux, True, dx, dy, gravity=G)
    assert device.fast_dry_ok(solver.store_of(p), eq)
    res = solver.step_patch(p, dt, eq, limiter, variant=_lib.VARIANT_FAST)
    want, cfl = O.step_2d(q, aux, dt, dx, dy, O.SWE2D, True, True, limiter, G)
    assert norm_rel(p.state, want) <= 1e-12, norm_rel(p.state, want)
    assert abs(res.max_courant - cfl) <= 1e-14 * max(cfl, 1.0)


def test_wet_dry_flag_rejected_for_other_forms():
    """ADJ_STEP_WET_DRY covers forward shallow water and its time-reversed
    f-wave adjoint; other forms on dry levels step with the EXACT kernel."""
    from paper_1511_03645_b200 import device, solver
    q, aux = dry_case(2, 40, 36)
    _, p = patch_from_arrays(q, aux, True, 1000.0, 1000.0, gravity=G)
    st = solver.store_of(p)
    st.sync_in()
    assert device.fast_dry_ok(st, make_equation("swe_adj_rev", gravity=G))
    assert device.fast_dry_ok(st, make_equation("swe_dry", gravity=G))
    from paper_1511_03645_b200 import equations as E
    from tests.helpers import dummy_model
    assert not device.fast_dry_ok(st, E.SweLinear2D(dummy_model("swe", G)).adjoint())   # f-wave, not reversed


def test_streamed_host_step_with_dry_cells():
    """step_patch_host on a level with dry cells (row slabs through the wet/dry
    march) equals the device step."""
    import torch
    from paper_1511_03645_b200 import _lib, solver
    q, aux = dry_case(7, 150, 120)
    dx = dy = 500.0
    dt = 0.8 * dx / float(np.max(aux[0]))
    eq = make_equation("swe_dry", gravity=G)
    bc = solver.BoundarySpec("wall", "outflow", "wall", "wall")
    _, p1 = patch_from_arrays(q, aux, True, dx, dy, gravity=G)
    _, p2 = patch_from_arrays(q, aux, True, dx, dy, gravity=G)
    host = torch.from_numpy(np.array(q, copy=True)).pin_memory()
    for _ in range(3):
        solver.fill_ghost_physical(p1, bc, eq, (150, 120))
        solver.step_patch(p1, dt, eq, "MC", variant=_lib.VARIANT_FAST)
        solver.step_patch_host(p2, host, dt, eq, bc, (150, 120), "MC", slabs=3)
    assert np.array_equal(host.numpy(), np.array(p1.state))


def test_job_classes_equal_wet_dry_march(monkeypatch):
    """Per-job classes (all-wet jobs without the selects, all-dry jobs copied)
    change no value against running every job through the wet/dry march."""
    from paper_1511_03645_b200 import _lib, device, solver
    outs = []
    for use in (False, True):
        monkeypatch.setattr(device, "USE_JOB_CLASS", use)
        q, aux = dry_case(9, 300, 260)
        dx = dy = 500.0
        dt = 0.8 * dx / float(np.max(aux[0]))
        eq = make_equation("swe_dry", gravity=G)
        _, p = patch_from_arrays(q, aux, True, dx, dy, gravity=G)
        bc = solver.BoundarySpec("wall", "wall", "wall", "wall")
        solver.advance_uniform(p, eq, bc, (300, 260), dt, 6, "MC", _lib.VARIANT_FAST)
        outs.append(np.array(p.state))
    assert np.array_equal(outs[0], outs[1])
