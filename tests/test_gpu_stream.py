"""solver.step_patch_host (row slabs streamed through the device with the
H2D copy, fill + step and D2H copy of consecutive slabs overlapping) equals
fill_ghost_physical + step_patch on the device, bitwise on the whole
ghost-inclusive state, for any slab count."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _per_cell_materials(monkeypatch):
    """These tests compare differently decomposed FAST runs bitwise.  With per-job
    materials (ADJ_STEP_UNIFORM_MAT) a cell is stepped by the invariant-material march or by
    the per-cell one depending on the job it falls in, and the two agree to rounding, not
    bitwise (tests/test_gpu_uniform_mat.py): the comparison pins the per-cell march, in this
    process and in spawned ranks."""
    from paper_1511_03645_b200 import device
    monkeypatch.setattr(device, "USE_UNIFORM_MAT", False)
    monkeypatch.setenv("ADJAMR_UNIFORM_MAT", "0")


def _patch(system, nx, ny, bc_sides):
    from paper_1511_03645_b200 import equations as E
    from paper_1511_03645_b200 import solver
    from paper_1511_03645_b200.geometry import Patch, PatchHierarchy
    if system == "swe":
        eq = E.SweLinear2D(E.SweMaterialModel(
            lambda x, y: -3000.0 + 800.0 * np.sin(3e-6 * x) * np.cos(2e-6 * y), 0.0, 9.81))
        xlim, ylim = (0.0, 1e6), (0.0, 9e5)
    else:
        eq = E.Acoustics2D(E.AcousticsMaterialModel(
            lambda x, y: 1.0 + 3.0 * (np.asarray(y) < 0.2 * np.asarray(x)),
            lambda x, y: np.where(np.asarray(y) < 0.2 * np.asarray(x), 1.0, 1.5)))
        xlim, ylim = (0.0, 1.0), (0.0, 0.9)
    h = PatchHierarchy(xlim=xlim, ylim=ylim, base_shape=(nx, ny), ratios=[])
    p = Patch(h.make_spec(1, (0, 0), (nx - 1, ny - 1)), 3)
    bc = solver.BoundarySpec(*bc_sides)
    solver.sample_patch_material(p, eq, bc, (nx, ny))
    rng = np.random.default_rng(3)
    cs = p.spec.cell_centers()
    X, Y = np.meshgrid(cs[0], cs[1], indexing="ij")
    sx, sy = xlim[1] - xlim[0], ylim[1] - ylim[0]
    p.interior()[0] = np.exp(-(((X - 0.4 * sx) / (0.05 * sx)) ** 2 + ((Y - 0.5 * sy) / (0.05 * sy)) ** 2))
    p.interior()[1] = 0.1 * rng.standard_normal((nx, ny))
    h.levels = [[p]]
    dt = solver.select_dt(h, eq, 0.9)
    return h, p, eq, bc, dt


@pytest.mark.parametrize("system", ["swe", "ac"])
@pytest.mark.parametrize("slabs", [1, 3, 7, 16])
def test_streamed_step_equals_device_step(system, slabs):
    import torch
    from paper_1511_03645_b200 import _lib, solver
    sides = ("wall", "outflow", "outflow", "wall")
    h, p, eq, bc, dt = _patch(system, 301, 263, sides)
    shape = (301, 263)
    start = np.array(p.state, copy=True)
    # reference path: device fill + step, full state downloaded
    want = []
    for _ in range(3):
        solver.fill_ghost_physical(p, bc, eq, shape)
        solver.step_patch(p, dt, eq, "MC", variant=_lib.VARIANT_FAST)
        want.append(np.array(p.state, copy=True))
    # streamed path on a pinned host state
    h2, p2, eq2, bc2, dt2 = _patch(system, 301, 263, sides)
    assert dt2 == dt and np.array_equal(np.array(p2.state), start)
    host = torch.from_numpy(start.copy()).pin_memory()
    for k in range(3):
        solver.step_patch_host(p2, host, dt, eq2, bc2, shape, "MC", slabs=slabs)
        assert np.array_equal(host.numpy(), want[k]), (k, float(np.abs(host.numpy() - want[k]).max()))
        assert np.array_equal(np.array(p2.state), want[k])
    assert p2.time == p.time


def test_streamed_step_raises_cfl_before_mutation():
    import torch
    from paper_1511_03645_b200 import solver
    h, p, eq, bc, dt = _patch("ac", 64, 48, ("outflow",) * 4)
    host = torch.from_numpy(np.array(p.state, copy=True)).pin_memory()
    before = host.clone()
    with pytest.raises(solver.CflViolationError):
        solver.step_patch_host(p, host, 3.0 * dt, eq, bc, (64, 48), "MC")
    assert torch.equal(host, before)


@pytest.mark.parametrize("slabs", [1, 5, 16])
def test_streamed_steps_without_wait_equal_waited_steps(slabs):
    """step_patch_host(wait=False): consecutive steps overlap their copies slab
    by slab; after host_stream_finish the host state equals the waited path's
    bitwise, and a non-finite value is still reported."""
    import torch
    from paper_1511_03645_b200 import solver
    sides = ("wall", "outflow", "outflow", "wall")
    shape = (301, 263)
    outs = []
    for wait in (True, False):
        h, p, eq, bc, dt = _patch("swe", *shape, sides)
        host = torch.from_numpy(np.array(p.state, copy=True)).pin_memory()
        for _ in range(5):
            solver.step_patch_host(p, host, dt, eq, bc, shape, "MC", slabs=slabs, wait=wait)
        solver.host_stream_finish(p)
        outs.append(host.numpy().copy())
        assert np.array_equal(np.array(p.state), outs[-1])
    assert np.array_equal(outs[0], outs[1])
    h, p, eq, bc, dt = _patch("ac", *shape, sides)
    q = np.array(p.state, copy=True)
    q[0, 40, 40] = np.nan
    host = torch.from_numpy(q).pin_memory()
    solver.step_patch_host(p, host, dt, eq, bc, shape, "MC", slabs=slabs, wait=False)
    solver.step_patch_host(p, host, dt, eq, bc, shape, "MC", slabs=slabs, wait=False)
    with pytest.raises(solver.NumericalBlowupError):
        solver.host_stream_finish(p)


def test_async_host_steps_then_device_steps_are_ordered():
    """Device steps issued after step_patch_host(wait=False) wait for its
    pending device-to-host copies (LevelStore.settle_pending): the host state
    after host_stream_finish is the async step's result, not a later one."""
    import torch
    from paper_1511_03645_b200 import _lib, solver
    sides = ("wall", "outflow", "outflow", "wall")
    shape = (301, 263)
    h, p, eq, bc, dt = _patch("ac", *shape, sides)
    h2, p2, eq2, bc2, _ = _patch("ac", *shape, sides)
    host = torch.from_numpy(np.array(p.state, copy=True)).pin_memory()
    solver.step_patch_host(p, host, dt, eq, bc, shape, "MC", slabs=4, wait=False)
    for _ in range(4):                       # device steps overwrite the store's buffers in rotation
        solver.fill_ghost_physical(p, bc, eq, shape)
        solver.step_patch(p, dt, eq, "MC", variant=_lib.VARIANT_FAST)
    solver.host_stream_finish(p)
    solver.fill_ghost_physical(p2, bc2, eq2, shape)
    solver.step_patch(p2, dt, eq2, "MC", variant=_lib.VARIANT_FAST)
    assert np.array_equal(host.numpy(), np.array(p2.state))
