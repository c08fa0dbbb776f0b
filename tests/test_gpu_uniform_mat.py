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


def _two_layer(nx, ny, seed):
    """BASELINE C3's medium on a small grid: K=4, rho=1 below y = 0.2 x, K=1, rho=1.5 above."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((3, nx + 4, ny + 4))
    xs = (np.arange(-2, nx + 2) + 0.5) / nx
    ys = (np.arange(-2, ny + 2) + 0.5) / ny
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    low = Y < 0.2 * X
    bulk = np.where(low, 4.0, 1.0)
    rho = np.where(low, 1.0, 1.5)
    c = np.sqrt(bulk / rho)
    aux = np.stack([c, rho * c, rho, bulk])
    eq = make_equation("ac2d")
    h, p = patch_from_arrays(q, aux, False, 1.0 / nx, 1.0 / ny)
    return h, p, eq, q, aux


@pytest.mark.parametrize("shape", [(300, 200), (140, 90)])
def test_per_job_material_on_a_two_layer_medium(shape):
    """Piecewise-constant medium: jobs whose strips read one material march
    with it as an invariant, the jobs crossing the interface per cell; equal to
    the all-per-cell run at 1e-13 and to the oracle at the FAST tolerance."""
    from paper_1511_03645_b200 import _lib, device, solver
    nx, ny = shape
    outs = []
    for on in (True, False):
        old = device.USE_UNIFORM_MAT
        device.USE_UNIFORM_MAT = on
        try:
            h, p, eq, q, aux = _two_layer(nx, ny, 4)
            st = solver.store_of(p)
            assert st.uniform_mat is None
            tiles, ntile, jobs, njob = st.tiles(_lib.VARIANT_FAST)
            ju = st.job_uniform(tiles, ntile, jobs, njob)
            if on:
                ju = ju.cpu().numpy().reshape(-1, 2)
                mats = {tuple(r) for r in ju.tolist()}
                assert (0.0, 0.0) in mats and len(mats) >= 2      # mixed jobs and single-material jobs
                assert mats <= {(0.0, 0.0), (2.0, 2.0), (float(aux[0].min()), float(aux[1].min()))}
            else:
                assert ju is None
            dt = 0.4 * min(p.spec.dx, p.spec.dy) / 2.0
            solver.step_patch(p, dt, eq, "MC", variant=_lib.VARIANT_FAST)
            outs.append(np.array(p.state, copy=True))
        finally:
            device.USE_UNIFORM_MAT = old
    assert norm_rel(outs[0], outs[1]) <= 1e-13
    want, _ = O.step_2d(q, aux, dt, 1.0 / nx, 1.0 / ny, O.AC2D, False, False, "MC")
    assert norm_rel(outs[0], want) <= 1e-12


def test_per_job_material_advance_uniform():
    """The in-launch physical fill (edge jobs first: a reordered job table) with per-job materials."""
    from paper_1511_03645_b200 import _lib, device, solver
    outs = []
    for on in (True, False):
        old = device.USE_UNIFORM_MAT
        device.USE_UNIFORM_MAT = on
        try:
            h, p, eq, q, aux = _two_layer(260, 120, 6)
            bc = solver.BoundarySpec("periodic", "periodic", "wall", "wall")
            dt = 0.45 * min(p.spec.dx, p.spec.dy) / 2.0
            solver.advance_uniform(p, eq, bc, (260, 120), dt, 9, "MC", _lib.VARIANT_FAST)
            outs.append(np.array(p.state, copy=True))
        finally:
            device.USE_UNIFORM_MAT = old
    assert norm_rel(outs[0], outs[1]) <= 1e-13


def test_streamed_and_sharded_steps_with_per_job_materials():
    """The decomposed paths (row slabs streamed from the host; x-slab shards)
    with per-job materials agree with the whole-level step to rounding."""
    import torch
    from paper_1511_03645_b200 import _lib, solver
    from tests.test_gpu_stream import _patch as stream_patch
    sides = ("wall", "outflow", "outflow", "wall")
    h, p, eq, bc, dt = stream_patch("ac", 301, 263, sides)
    start = np.array(p.state, copy=True)
    for _ in range(3):
        solver.fill_ghost_physical(p, bc, eq, (301, 263))
        solver.step_patch(p, dt, eq, "MC", variant=_lib.VARIANT_FAST)
    h2, p2, eq2, bc2, _ = stream_patch("ac", 301, 263, sides)
    host = torch.from_numpy(start.copy()).pin_memory()
    for _ in range(3):
        solver.step_patch_host(p2, host, dt, eq2, bc2, (301, 263), "MC", slabs=5)
    assert norm_rel(host.numpy()[:, 2:-2, 2:-2], np.array(p.state)[:, 2:-2, 2:-2]) <= 1e-13


def test_per_job_material_over_several_patches():
    """A level of 32^2 patches, each with its own constant material and one
    with a varying one: short strips of different patches share warp jobs, so a
    packed job is single-material only when all its strips agree.  Every patch
    equals its own oracle step and the per-cell run."""
    from paper_1511_03645_b200 import _lib, device, solver
    rng = np.random.default_rng(11)
    mats = [(2.0, 2.0), (2.0, 2.0), (1.25, 1.5), (2.0, 2.0), None, (1.25, 1.5), (2.0, 2.0), (2.0, 2.0)]
    nx = ny = 32
    dx = dy = 1.0 / 256
    qs, auxs = [], []
    for m in mats:
        qs.append(rng.standard_normal((3, nx + 4, ny + 4)))
        if m is None:
            rho = rng.uniform(0.8, 1.5, (nx + 4, ny + 4))
            bulk = rng.uniform(1.0, 4.0, (nx + 4, ny + 4))
            c = np.sqrt(bulk / rho)
            auxs.append(np.stack([c, rho * c, rho, bulk]))
        else:
            c, z = m
            auxs.append(np.stack([np.full((nx + 4, ny + 4), v) for v in (c, z, z / c, z * c)]))
    eq = make_equation("ac2d")
    dt = 0.4 * dx / 2.3
    outs = []
    for on in (True, False):
        old = device.USE_UNIFORM_MAT
        device.USE_UNIFORM_MAT = on
        try:
            ps = [patch_from_arrays(q, a, False, dx, dy, lo=(32 * k, 0))[1] for k, (q, a) in enumerate(zip(qs, auxs))]
            st = device.LevelStore(ps)
            assert st.uniform_mat is None
            st.sync_in()
            tiles, ntile, jobs, njob = st.tiles(_lib.VARIANT_FAST)
            ju = st.job_uniform(tiles, ntile, jobs, njob)
            if on:
                ju = ju.cpu().numpy().reshape(-1, 2)
                offs = jobs.cpu().numpy()
                rows = np.frombuffer(tiles.cpu().numpy().tobytes(), dtype=_lib.TILE_DTYPE)[:ntile]
                for j in range(njob):               # a job is single-material iff all its strips' patches agree
                    want = {mats[int(r["patch"])] for r in rows[offs[j]:offs[j + 1]]}
                    assert tuple(ju[j]) == (want.pop() if len(want) == 1 and None not in want else (0.0, 0.0))
                assert any(offs[j + 1] - offs[j] > 1 and ju[j, 0] == 0.0 for j in range(njob))   # a mixed packed job
            out = st._free(st.cur)
            device.launch_step(st, dt, eq, "MC", _lib.VARIANT_FAST, out, accumulate=True)
            st.cur = out
            res = [st.view(k).cpu().numpy().copy() for k in range(len(ps))]
            outs.append(res)
        finally:
            device.USE_UNIFORM_MAT = old
    for k, (q, a) in enumerate(zip(qs, auxs)):
        want, _ = O.step_2d(q, a, dt, dx, dy, O.AC2D, False, False, "MC")
        got_on, got_off = outs[0][k][:, 2:-2, 2:-2], outs[1][k][:, 2:-2, 2:-2]
        assert norm_rel(got_on, got_off) <= 1e-13
        assert norm_rel(got_on, want[:, 2:-2, 2:-2]) <= 1e-12


def test_job_classification_skipped_on_levels_of_many_patches():
    from paper_1511_03645_b200 import _lib, device
    rng = np.random.default_rng(2)
    ps = []
    for k in range(device.LevelStore.JOB_UNIFORM_MAX_PATCHES + 1):
        aux = np.stack([np.full((20, 20), v) for v in ((2.0, 2.0, 1.0, 4.0) if k else (1.0, 1.0, 1.0, 1.0))])
        ps.append(patch_from_arrays(rng.standard_normal((3, 20, 20)), aux, False, 0.1, 0.1, lo=(16 * k, 0))[1])
    st = device.LevelStore(ps)
    assert st.uniform_mat is None
    assert st.job_uniform(*st.tiles(_lib.VARIANT_FAST)) is None
