"""Host-side AMR bookkeeping vs the reference's golden outputs (CPU only)."""
import numpy as np
import pytest

from paper_1511_03645_b200 import amr
from paper_1511_03645_b200.geometry import Patch, PatchHierarchy, allowed_region_mask
from tests.golden_io import load

H = load("host.npz")
CL = sorted(k for k in H if k.startswith("c"))


@pytest.mark.parametrize("case", CL)
def test_cluster_buffer_rectangles(case):
    d = H[case]
    mask = d["mask"].astype(bool)
    nd = mask.ndim
    me = None if d["max_edge"] < 0 else int(d["max_edge"])
    boxes = amr.cluster(mask, float(d["eff"]), max_edge=me)
    got = np.array([[*b.lo, *b.hi, b.efficiency] for b in boxes], dtype=float).reshape(-1, 2 * nd + 1)
    assert np.array_equal(got, d["boxes"])
    ff = amr.FlagField(flags=mask, lo=(0,) * nd, level=1, strategy_name="x", time=0.0)
    assert np.array_equal(amr.buffer_flags(ff, int(d["buf"])).flags, d["buffered"])
    allowed = d["allowed"].astype(bool)
    rects = []
    for b in boxes:
        rects += amr._allowed_rectangles(b, allowed, mask & allowed)
    got = np.array([[*b.lo, *b.hi, b.efficiency] for b in rects], dtype=float).reshape(-1, 2 * nd + 1)
    assert np.array_equal(got, d["rects"])


@pytest.mark.parametrize("case", sorted(k for k in H if k.startswith("n")))
def test_allowed_region(case):
    d = H[case]
    h = PatchHierarchy(xlim=(0, 1), ylim=(0, 1), base_shape=(16, 12), ratios=[2])
    h.levels = [[Patch(h.make_spec(1, tuple(b[:2]), tuple(b[2:])), 3) for b in d["boxes"].reshape(-1, 4)]]
    assert np.array_equal(allowed_region_mask(h, 1), d["allowed"])


def test_ghost_rect_cover_is_exact():
    """Ghost rectangles of a level cover each in-domain ghost cell exactly once
    per source kind (same-level sources are disjoint interiors)."""
    h = PatchHierarchy(xlim=(0, 1), ylim=(0, 1), base_shape=(8, 8), ratios=[2])
    coarse = [Patch(h.make_spec(1, (0, 0), (7, 7)), 3)]
    fine = [Patch(h.make_spec(2, lo, hi), 3) for lo, hi in [((2, 2), (7, 9)), ((8, 2), (13, 5)), ((8, 6), (11, 11))]]
    h.levels = [coarse, fine]
    crects, copies, covered = amr.build_ghost_rects(h, 2)
    for k, p in enumerate(fine):
        ring, phys = amr._ring_and_physical(p.spec, h.level_shape(2))
        assert covered[k] + phys == ring
    seen = {}
    for r in copies:
        key = r[1]
        for i in range(r[5]):
            for j in range(r[6]):
                cell = (key, r[3] + i, r[4] + j)
                assert cell not in seen
                seen[cell] = 1


@pytest.mark.parametrize("case", CL)
def test_native_and_python_clustering_agree_with_reference(case):
    d = H[case]
    mask = d["mask"].astype(bool)
    nd = mask.ndim
    me = None if d["max_edge"] < 0 else int(d["max_edge"])
    for native in (True, False):
        boxes = amr.cluster(mask, float(d["eff"]), max_edge=me, native=native)
        got = np.array([[*b.lo, *b.hi, b.efficiency] for b in boxes], dtype=float).reshape(-1, 2 * nd + 1)
        assert np.array_equal(got, d["boxes"]), native


def test_native_clustering_matches_python_on_large_masks():
    rng = np.random.default_rng(11)
    for n, cover, me in ((300, 0.2, 12), (512, 0.35, 30), (257, 0.5, None)):
        yy, xx = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        m = np.zeros((n, n), bool)
        while m.mean() < cover:
            cx, cy = rng.uniform(0, n, 2)
            r = rng.uniform(3, n / 8)
            m |= (xx - cx) ** 2 + (yy - cy) ** 2 <= r * r
        m ^= rng.random((n, n)) < 0.01
        a = amr.cluster(m, 0.7, max_edge=me, native=True)
        b = amr.cluster(m, 0.7, max_edge=me, native=False)
        assert [(x.lo, x.hi, x.efficiency) for x in a] == [(x.lo, x.hi, x.efficiency) for x in b]


def _random_hierarchy(rng, nd):
    """Coarse level tiled into boxes, fine level from clustering a random blob
    mask (disjoint boxes), some touching the domain edge."""
    if nd == 2:
        h = PatchHierarchy(xlim=(0, 1), ylim=(0, 1), base_shape=(24, 20), ratios=[2])
        coarse = [Patch(h.make_spec(1, (x, y), (min(x + 7, 23), min(y + 9, 19))), 3)
                  for x in range(0, 24, 8) for y in range(0, 20, 10)]
        mask = np.zeros((48, 40), dtype=bool)
        for _ in range(6):
            cx, cy, r = rng.integers(0, 48), rng.integers(0, 40), rng.integers(2, 9)
            X, Y = np.meshgrid(np.arange(48), np.arange(40), indexing="ij")
            mask |= (X - cx) ** 2 + (Y - cy) ** 2 < r * r
    else:
        h = PatchHierarchy(xlim=(0, 1), ylim=None, base_shape=(40,), ratios=[2])
        coarse = [Patch(h.make_spec(1, (x,), (min(x + 9, 39),)), 2) for x in range(0, 40, 10)]
        mask = rng.random(80) < 0.3
    boxes = amr.cluster(mask, 0.7, max_edge=12)
    fine = [Patch(h.make_spec(2, b.lo, b.hi), 3 if nd == 2 else 2) for b in boxes]
    h.levels = [coarse, fine]
    return h


@pytest.mark.parametrize("nd", [1, 2])
def test_native_ghost_rects_equal_python(nd):
    rng = np.random.default_rng(7 + nd)
    for _ in range(8):
        h = _random_hierarchy(rng, nd)
        for level in (1, 2):
            for disjoint in (False, True):
                for only in (None, h.patches(level)[len(h.patches(level)) // 2]):
                    a = amr.build_ghost_rects(h, level, only=only, disjoint=disjoint, native=True)
                    b = amr.build_ghost_rects(h, level, only=only, disjoint=disjoint, native=False)
                    assert a[0] == b[0]
                    assert a[1] == b[1]
                    assert np.array_equal(a[2], b[2])
