"""Host-side AMR bookkeeping vs the reference's golden outputs (CPU only)."""
import numpy as np
import pytest

from paper_1511_03645_b200 import _lib, amr
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


@pytest.mark.parametrize("nd", [1, 2])
def test_native_box_overlaps_equal_python_scan(nd):
    """adj_box_overlaps gives the rects (and order) of the per-patch scan of
    the regrid fill (amr.py:504-551): parents refined by the ratio (COARSE)
    and old patches (COPY)."""
    rng = np.random.default_rng(11 + nd)
    for _ in range(6):
        h = _random_hierarchy(rng, nd)
        parents, new = h.patches(1), h.patches(2)
        g = new[0].spec.ghost_width
        r = h.ratio_to_finer(1)
        got = amr._box_overlaps(_lib.RECT_COARSE, new, parents, g, g, r).tolist()
        c_lo, c_hi = amr._boxes(parents)
        cf_lo, cf_hi = c_lo * r, (c_hi + 1) * r - 1
        want = []
        for k, p in enumerate(new):
            for c in amr._candidates(cf_lo, cf_hi, p.spec.lo, p.spec.hi):
                ib = amr._intersect(p.spec.lo, p.spec.hi, tuple(cf_lo[c]), tuple(cf_hi[c]))
                if ib is not None:
                    ext = [hh - ll + 1 for ll, hh in zip(*ib)]
                    want.append(amr._rect(_lib.RECT_COARSE, k, int(c), ib[0], p.spec, ext))
        assert got == want
        old = [Patch(h.make_spec(2, b.lo, b.hi), 3 if nd == 2 else 2)
               for b in amr.cluster(rng.random(tuple(h.level_shape(2))) < 0.2, 0.6, max_edge=10)]
        got = amr._box_overlaps(_lib.RECT_COPY, new, old, g, g, 1).tolist()
        o_lo, o_hi = amr._boxes(old)
        want = []
        for k, p in enumerate(new):
            for o in amr._candidates(o_lo, o_hi, p.spec.lo, p.spec.hi):
                ib = amr._intersect(p.spec.lo, p.spec.hi, tuple(o_lo[o]), tuple(o_hi[o]))
                if ib is not None:
                    ext = [hh - ll + 1 for ll, hh in zip(*ib)]
                    want.append(amr._rect(_lib.RECT_COPY, k, int(o), ib[0], p.spec, ext, ib[0], old[o].spec))
        assert got == want


def test_batched_material_sampling_equals_per_patch():
    """solver.sample_patches_material (one model call on stacked cell
    centres) gives each patch exactly sample_patch_material's aux,
    including wall / outflow ghost treatment (solver.py:180-205)."""
    from paper_1511_03645_b200 import equations as E, solver
    h = PatchHierarchy(xlim=(0.0, 1.0), ylim=(0.0, 1.0), base_shape=(64, 64), ratios=[2])
    bc = solver.BoundarySpec("wall", "outflow", "wall", "outflow")
    eqs = (E.Acoustics2D(E.AcousticsMaterialModel(lambda x, y: 1.0 + 3.0 * (np.asarray(y) < 0.2 * np.asarray(x)),
                                                  lambda x, y: np.where(np.asarray(y) < 0.2 * np.asarray(x), 1.0, 1.5))),
           E.SweLinear2D(E.SweMaterialModel(lambda x, y: -50.0 + 80.0 * np.sin(3 * np.asarray(x)) * np.cos(2 * np.asarray(y)),
                                            0.0, 9.81)))
    boxes = [((0, 32 * k), (31, 32 * k + 31)) for k in range(4)] + [((96, 32 * k), (127, 32 * k + 31)) for k in range(4)]
    # regrid clusters come in mixed shapes: one flattened call covers them all
    mixed = [((0, 0), (15, 47)), ((16, 0), (63, 7)), ((64, 64), (127, 127)), ((40, 100), (41, 127)), ((0, 120), (3, 127))]
    for eq in eqs:
        a = [Patch(h.make_spec(2, lo, hi), 3) for lo, hi in mixed]
        b = [Patch(h.make_spec(2, lo, hi), 3) for lo, hi in mixed]
        solver.sample_patches_material(a, eq, bc, (128, 128))
        for p in b:
            solver.sample_patch_material(p, eq, bc, (128, 128))
        for pa, pb in zip(a, b):
            for x, y in zip(pa.aux.planes(), pb.aux.planes()):
                assert np.array_equal(x, y)
    for eq in eqs:
        a = [Patch(h.make_spec(2, lo, hi), 3) for lo, hi in boxes]
        b = [Patch(h.make_spec(2, lo, hi), 3) for lo, hi in boxes]
        solver.sample_patches_material(a, eq, bc, (128, 128))
        for p in b:
            solver.sample_patch_material(p, eq, bc, (128, 128))
        for pa, pb in zip(a, b):
            assert type(pa.aux) is type(pb.aux)
            for x, y in zip(pa.aux.planes(), pb.aux.planes()):
                assert np.array_equal(x, y)
    # a non-elementwise model falls back to per-patch calls
    shape_dependent = E.Acoustics2D(E.AcousticsMaterialModel(lambda x, y: np.full(np.shape(x), 2.0 + np.asarray(x).ndim),
                                                             lambda x, y: np.ones_like(np.asarray(x, float))))
    a = [Patch(h.make_spec(2, lo, hi), 3) for lo, hi in boxes]
    solver.sample_patches_material(a, shape_dependent, bc, (128, 128))
    assert np.all(a[0].aux.bulk == 4.0)
