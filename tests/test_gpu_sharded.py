"""Sharded uniform level on the device: x-slabs stepped with
the halo exchange (sharded.advance_local_shards: several slabs in one
process; sharded.advance_sharded at world size 1) equal the unsharded
advance_uniform run bitwise on every interior cell, for shallow water and
heterogeneous acoustics with wall and outflow sides."""
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


def _eq_geom(system):
    from paper_1511_03645_b200 import equations as E
    if system == "swe":
        eq = E.SweLinear2D(E.SweMaterialModel(
            lambda x, y: -3000.0 + 800.0 * np.sin(3e-6 * x) * np.cos(2e-6 * y), 0.0, 9.81))
        return eq, (0.0, 1e6), (0.0, 9e5)
    eq = E.Acoustics2D(E.AcousticsMaterialModel(
        lambda x, y: 1.0 + 3.0 * (np.asarray(y) < 0.2 * np.asarray(x)),
        lambda x, y: np.where(np.asarray(y) < 0.2 * np.asarray(x), 1.0, 1.5)))
    return eq, (0.0, 1.0), (0.0, 0.9)


def _init(p, xlim, ylim):
    cs = p.spec.cell_centers()
    X, Y = np.meshgrid(cs[0], cs[1], indexing="ij")
    sx, sy = xlim[1] - xlim[0], ylim[1] - ylim[0]
    p.interior()[0] = np.exp(-(((X - 0.4 * sx) / (0.05 * sx)) ** 2 + ((Y - 0.5 * sy) / (0.05 * sy)) ** 2))
    p.interior()[1] = 0.1 * np.sin(X / sx * 7.0) * np.cos(Y / sy * 5.0)


def _setup(system, nx, ny, sides, world):
    from paper_1511_03645_b200 import solver
    from paper_1511_03645_b200.geometry import Patch, PatchHierarchy
    from paper_1511_03645_b200.sharded import shard_patch
    eq, xlim, ylim = _eq_geom(system)
    h = PatchHierarchy(xlim=xlim, ylim=ylim, base_shape=(nx, ny), ratios=[])
    bc = solver.BoundarySpec(*sides)
    whole = Patch(h.make_spec(1, (0, 0), (nx - 1, ny - 1)), 3)
    solver.sample_patch_material(whole, eq, bc, (nx, ny))
    _init(whole, xlim, ylim)
    h.levels = [[whole]]
    dt = solver.select_dt(h, eq, 0.9)
    shards = []
    for r in range(world):
        # same material and initial values as the whole patch's window (recomputing cell
        # centres from the slab origin would round differently)
        p = shard_patch(h, r, world, 3)
        x0, x1 = p.spec.lo[0], p.spec.hi[0] + 1
        p.aux = whole.aux[(slice(x0, x1 + 4), slice(None))]
        p.state = np.array(np.asarray(whole.state)[:, x0:x1 + 4], copy=True)
        shards.append(p)
    return h, whole, shards, eq, bc, dt


@pytest.mark.parametrize("variant", ["exact", "fast"])
@pytest.mark.parametrize("system", ["swe", "ac"])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_local_shards_equal_unsharded(system, world, variant):
    """EXACT: bitwise.  FAST: within its 1e-12 norm-relative tolerance (a slab
    boundary can shift which register-ring column body computes a cell)."""
    from paper_1511_03645_b200 import _lib, solver
    from paper_1511_03645_b200.sharded import advance_local_shards
    from tests.helpers import norm_rel
    var = _lib.VARIANT_EXACT if variant == "exact" else _lib.VARIANT_FAST
    sides = ("wall", "outflow", "outflow", "wall")
    nx, ny = 157, 133
    h, whole, shards, eq, bc, dt = _setup(system, nx, ny, sides, world)
    solver.advance_uniform(whole, eq, bc, (nx, ny), dt, 7, "MC", var, graph=False)
    want = np.array(whole.state)[:, 2:-2, 2:-2]
    advance_local_shards(shards, eq, bc, (nx, ny), dt, 7, "MC", var)
    for p in shards:
        x0, x1 = p.spec.lo[0], p.spec.hi[0] + 1
        got = np.array(p.state)[:, 2:-2, 2:-2]
        if variant == "exact":
            assert np.array_equal(got, want[:, x0:x1]), (x0, float(np.abs(got - want[:, x0:x1]).max()))
        else:
            assert norm_rel(got, want[:, x0:x1]) <= 1e-12
        assert p.time == whole.time


def test_sharded_world1_equals_uniform():
    from paper_1511_03645_b200 import _lib, solver
    from paper_1511_03645_b200.sharded import DistTransport, advance_sharded
    sides = ("outflow",) * 4
    h, whole, shards, eq, bc, dt = _setup("swe", 140, 128, sides, 1)
    solver.advance_uniform(whole, eq, bc, (140, 128), dt, 5, "MC", _lib.VARIANT_FAST, graph=False)
    advance_sharded(shards[0], eq, bc, (140, 128), dt, 5, DistTransport(0, 1), "MC", _lib.VARIANT_FAST)
    assert np.array_equal(np.array(shards[0].state)[:, 2:-2, 2:-2], np.array(whole.state)[:, 2:-2, 2:-2])


@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_sharded_graph_replay_equals_eager(variant):
    """advance_sharded with CUDA-graph step pairs (fill + fold + pack /
    unpack + K1 around the exchange) equals the eager loop bitwise, across
    calls of odd lengths (parity realignment)."""
    from paper_1511_03645_b200 import _lib
    from paper_1511_03645_b200.sharded import DistTransport, advance_sharded
    var = _lib.VARIANT_EXACT if variant == "exact" else _lib.VARIANT_FAST
    sides = ("wall", "outflow", "outflow", "wall")
    out = []
    for graph in (False, True):
        h, whole, shards, eq, bc, dt = _setup("ac", 96, 128, sides, 1)
        for n in (5, 4, 3):
            advance_sharded(shards[0], eq, bc, (96, 128), dt, n, DistTransport(0, 1), "MC", var, graph=graph)
        out.append(np.array(shards[0].state)[:, 2:-2, 2:-2])
        assert shards[0].time == pytest.approx(12 * dt)
    assert np.array_equal(out[0], out[1])
