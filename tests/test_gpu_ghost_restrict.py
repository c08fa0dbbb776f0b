"""K2 (physical, coarse->fine) and K4 (restriction) on the GPU vs the
reference's golden vectors (bitwise)."""
import numpy as np
import pytest

from tests.golden_io import load
from tests.helpers import material_from_planes

GHOST = load("ghost.npz")
RESTRICT = load("restrict.npz")
pytestmark = pytest.mark.gpu


def _ac_aux(shape):
    from paper_1511_03645_b200 import equations as E
    one = np.ones(shape)
    return E.AcousticsMaterial(bulk=one, rho=one, c=one, z=one)


@pytest.mark.parametrize("case", [c for c in sorted(GHOST) if c.startswith("phys")])
def test_physical_fill_bitwise(case):
    from paper_1511_03645_b200 import equations as E
    from paper_1511_03645_b200 import solver
    from paper_1511_03645_b200.geometry import Patch, PatchHierarchy
    d = GHOST[case]
    lo, shape, ls = tuple(d["lo"]), tuple(d["shape"]), tuple(d["level_shape"])
    h = PatchHierarchy(xlim=(0, 1), ylim=(0, 1), base_shape=ls, ratios=[])
    p = Patch(h.make_spec(1, lo, tuple(l + n - 1 for l, n in zip(lo, shape))), 3)
    p.aux = _ac_aux(d["q_in"].shape[1:])
    p.state = d["q_in"]
    bc = solver.BoundarySpec(*[str(s) for s in d["bc"]])
    eq = E.Acoustics2D(E.AcousticsMaterialModel(None, None))
    solver.fill_ghost_physical(p, bc, eq, ls)
    assert np.array_equal(p.state, d["q_out"])


def test_coarse_interp_bitwise():
    from paper_1511_03645_b200 import solver
    from paper_1511_03645_b200.geometry import Patch, PatchHierarchy
    d = GHOST["coarse0"]
    h = PatchHierarchy(xlim=(0.0, 2.0), ylim=(0.0, 1.5), base_shape=(16, 12), ratios=[2])
    cps = []
    for (lo, hi), old, new in ((((0, 0), (7, 11)), d["c0_old"], d["c0_new"]),
                               (((8, 0), (15, 11)), d["c1_old"], d["c1_new"])):
        cp = Patch(h.make_spec(1, lo, hi), 3)
        cp.aux = _ac_aux(old.shape[1:])
        cp.state = old
        cp.save_old()
        cp.time = 0.4
        cp.state = new
        cps.append(cp)
    fp = Patch(h.make_spec(2, (10, 6), (21, 17)), 3)
    fp.aux = _ac_aux((16, 16))
    h.levels = [cps, [fp]]
    g = 2
    ii, jj = np.meshgrid(np.arange(10 - g, 22 + g), np.arange(6 - g, 18 + g), indexing="ij")
    ghost = ~((ii >= 10) & (ii <= 21) & (jj >= 6) & (jj <= 17))
    indom = ghost & (ii >= 0) & (ii < 32) & (jj >= 0) & (jj < 24)
    for n, t in enumerate(d["t_list"]):
        fp.state = np.zeros((3, 16, 16))
        solver.fill_ghost_from_coarse(fp, h, float(t))
        assert np.array_equal(fp.state[:, indom], d[f"f_t{n}"][:, indom]), t
    with pytest.raises(solver.SchedulingError):
        solver.fill_ghost_from_coarse(fp, h, 2.0)


@pytest.mark.parametrize("case", sorted(RESTRICT))
def test_restrict_bitwise(case):
    from paper_1511_03645_b200 import amr
    from paper_1511_03645_b200.geometry import Patch, PatchHierarchy
    d = RESTRICT[case]
    r = int(d["ratio"])
    swe = str(d["name"]).startswith("swe")
    h = PatchHierarchy(xlim=(0.0, 1.2), ylim=(0.0, 1.0), base_shape=(12, 10), ratios=[r])
    cp = Patch(h.make_spec(1, (0, 0), (11, 9)), 3)
    cp.aux = material_from_planes(d["c_aux"], swe)
    cp.state = d["c_in"]
    fps = []
    for k in (0, 1):
        lohi = d["f_lohi"][k]
        fp = Patch(h.make_spec(2, tuple(lohi[:2]), tuple(lohi[2:])), 3)
        fp.aux = material_from_planes(d[f"f{k}_aux"], swe)
        fp.state = d[f"f{k}"]
        fps.append(fp)
    h.levels = [[cp], fps]
    amr.restrict_fine_to_coarse(h, 1)
    assert np.array_equal(cp.state, d["c_out"])
