"""K3 kernel layouts against the oracle (bitwise) on a multi-patch
shallow-water level with dry forward and dry adjoint cells, in both window
modes (adjoint.py:227-257, adjoint.py:98-110 for mode 1): the row-layout
kernel for single snapshots (every patch row a multiple of 128 cells), the
one-cell-per-lane kernel (ragged rows) and the pair kernel (windows of >= 2
snapshots)."""
import numpy as np
import pytest

from oracle import adjamr_oracle as O

pytestmark = pytest.mark.gpu

TIMES = np.linspace(0.0, 1.0, 6)
NXA = 48


def _level(shapes_los, seed):
    from paper_1511_03645_b200 import equations as E
    from paper_1511_03645_b200.geometry import Patch, PatchHierarchy
    rng = np.random.default_rng(seed)
    h = PatchHierarchy(xlim=(0.0, 1.0), ylim=(0.0, 1.0), base_shape=(64, 512), ratios=[])
    patches = []
    for lo, shape in shapes_los:
        spec = h.make_spec(1, lo, (lo[0] + shape[0] - 1, lo[1] + shape[1] - 1))
        p = Patch(spec, 3)
        G = (shape[0] + 4, shape[1] + 4)
        depth = rng.uniform(-0.3, 1.0, G)
        depth[depth < 0] = 0.0
        p.aux = E.SweMaterial(bathymetry=-depth, depth=depth, wet=depth > 0, c=np.sqrt(9.81 * depth), gravity=9.81)
        p.state = rng.standard_normal((3,) + G)
        patches.append(p)
    return h, patches


def _store(seed, dry, NYA):
    from paper_1511_03645_b200 import adjoint
    from paper_1511_03645_b200.geometry import UniformField
    rng = np.random.default_rng(seed)
    vals = rng.standard_normal((len(TIMES), 3, NXA, NYA))
    fields = [UniformField(values=vals[k], origin=(0.0, 0.0), dx=1.0 / NXA, dy=1.0 / NYA, time=t)
              for k, t in enumerate(TIMES)]
    wet = rng.uniform(size=(NXA, NYA)) > 0.1 if dry else None
    return vals, wet, adjoint.AdjointSnapshotStore(times=TIMES, fields=fields, window=adjoint.TimeWindow(0.0, 1.0),
                                                   wet=wet)


def _oracle(p, vals, wet, t, window, interp, NYA):
    from paper_1511_03645_b200 import adjoint
    lo, shape, dx, dy = p.spec.lo, p.spec.shape, p.spec.dx, p.spec.dy
    x = (np.arange(lo[0], lo[0] + shape[0]) + 0.5) * dx
    y = (np.arange(lo[1], lo[1] + shape[1]) + 0.5) * dy
    xc, yc = np.broadcast_to(x[:, None], shape), np.broadcast_to(y[None, :], shape)
    qi = p.state[:, 2:-2, 2:-2]
    fwd_wet = p.aux.wet[2:-2, 2:-2]
    if not interp:
        idx = adjoint.query_window_times(t, window, _FakeStore(window))
        return O.inner_product(qi, xc, yc, vals, idx, (0.0, 0.0), 1.0 / NXA, 1.0 / NYA, fwd_wet, wet), len(idx)
    upper = min(t + window.span, window.t_final)
    t_eval = [t] + [float(s) for s in TIMES if t + 1e-9 < s < upper - 1e-9] + ([upper] if upper > t + 1e-9 else [])
    best = O.inner_product_interp(qi, xc, yc, vals, TIMES, t_eval, (0.0, 0.0), 1.0 / NXA, 1.0 / NYA)
    best = np.where(fwd_wet, best, 0.0)
    if wet is not None:
        i = np.clip((xc / (1.0 / NXA)).astype(int), 0, NXA - 1)
        j = np.clip((yc / (1.0 / NYA)).astype(int), 0, NYA - 1)
        best = np.where(~wet[i, j], 0.0, best)
    return best, len(t_eval)


class _FakeStore:
    """query_window_times needs only times and the window."""
    def __init__(self, window):
        self.times = TIMES
        self.window = window


ROWS = [((0, 0), (20, 256)), ((20, 256), (17, 128)), ((40, 0), (8, 384))]
RAGGED = [((0, 0), (20, 250)), ((20, 256), (17, 100)), ((40, 0), (8, 33))]


# adjoint widths: a 128-cell segment spans ~27 (100 columns) or ~102 (400)
# adjoint columns; 128 columns = ratio 4, where every even-aligned column pair
# shares its stencil column (the paired row kernel, k3_rowp)
@pytest.mark.parametrize("layout,nya", [("rows", 100), ("rows", 400), ("rows", 128), ("ragged", 100)])
@pytest.mark.parametrize("interp", [False, True])
@pytest.mark.parametrize("case", ["snapshot", "between", "span"])
def test_layouts_bitwise(layout, nya, interp, case):
    from paper_1511_03645_b200 import adjoint
    _, patches = _level(ROWS if layout == "rows" else RAGGED, seed=3)
    vals, wet, store = _store(seed=4, dry=True, NYA=nya)
    t, window = {"snapshot": (0.6, adjoint.TimeWindow(0.6, 0.6)),
                 "between": (0.5, adjoint.TimeWindow(0.5, 0.5)),
                 "span": (0.3, adjoint.TimeWindow(0.0, 0.75))}[case]
    tol = 0.7
    flags, counts, best = adjoint.flag_level(patches, t, store, window, tol, want_best=True, time_interp=interp)
    for p, f, c, b in zip(patches, flags, counts, best):
        ref, n = _oracle(p, vals, wet, t, window, interp, nya)
        if case != "span":
            assert n == 1 or not interp and case == "between"
        assert np.array_equal(b, ref)
        assert np.array_equal(f, ref > tol)
        assert c == int((ref > tol).sum())


@pytest.mark.parametrize("nya,expect", [(128, True), (100, False), (256, False)])
def test_pair_layout_detection(nya, expect):
    """ADJ_FLAG_PAIRS is set exactly when every even-aligned column pair shares
    its adjoint stencil column (ratio 4 yes; ratio 2 pairs straddle a centre)."""
    from paper_1511_03645_b200 import adjoint, device, solver
    _, patches = _level(ROWS, seed=3)
    _, _, store = _store(seed=4, dry=False, NYA=nya)
    adjoint.flag_level(patches, 0.6, store, adjoint.TimeWindow(0.6, 0.6), 0.7)
    st = solver.store_of(patches[0])
    tabs = device.flag_axis_tables(st, (NXA, nya), (0.0, 0.0), 1.0 / NXA, 1.0 / nya, (0.0, 0.0),
                                   patches[0].spec.dx, patches[0].spec.dy)
    assert tabs[4] is expect
    assert tabs[5] is False      # 48 adjoint rows over 64 forward rows: row pairs straddle centres
    assert tabs[6] is False


@pytest.mark.parametrize("layout,nya", [("rows", 100), ("rows", 128), ("ragged", 100)])
@pytest.mark.parametrize("interp", [False, True])
def test_fast_variant_multi_snapshot(layout, nya, interp):
    """VARIANT_FAST (corner weights + FMAs) on a multi-snapshot window: inner
    products within 1e-12 norm-relative of the reference, flags identical
    except for cells within 1e-12 relative of the tolerance (north_star)."""
    from paper_1511_03645_b200 import _lib, adjoint
    _, patches = _level(ROWS if layout == "rows" else RAGGED, seed=5)
    vals, wet, store = _store(seed=6, dry=True, NYA=nya)
    t, window = 0.3, adjoint.TimeWindow(0.0, 0.75)
    tol = 0.7
    flags, counts, best = adjoint.flag_level(patches, t, store, window, tol, want_best=True, time_interp=interp,
                                             variant=_lib.VARIANT_FAST)
    for p, f, c, b in zip(patches, flags, counts, best):
        ref, n = _oracle(p, vals, wet, t, window, interp, nya)
        assert n >= 2
        assert np.max(np.abs(b - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1e-300)
        far = np.abs(ref - tol) > 1e-12 * tol
        assert np.array_equal(f[far], (ref > tol)[far])
        assert c == int(f.sum())


def _store_n(seed, nxa, nya, dry):
    from paper_1511_03645_b200 import adjoint
    from paper_1511_03645_b200.geometry import UniformField
    rng = np.random.default_rng(seed)
    vals = rng.standard_normal((len(TIMES), 3, nxa, nya))
    fields = [UniformField(values=vals[k], origin=(0.0, 0.0), dx=1.0 / nxa, dy=1.0 / nya, time=t)
              for k, t in enumerate(TIMES)]
    wet = rng.uniform(size=(nxa, nya)) > 0.1 if dry else None
    return vals, wet, adjoint.AdjointSnapshotStore(times=TIMES, fields=fields, window=adjoint.TimeWindow(0.0, 1.0),
                                                   wet=wet)


@pytest.mark.parametrize("variant", ["exact", "fast"])
@pytest.mark.parametrize("dry", [False, True])
def test_quad_kernel_multi_snapshot(variant, dry):
    """Ratio 4 in both axes (adjoint 16 x 128 under the 64 x 512 level): every
    even-aligned 2x2 quad shares its stencil, so windows of >= 2 snapshots run
    the quad kernel (k3_quad).  EXACT: bitwise; FAST: 1e-12 norm-relative and
    flags equal away from the tolerance."""
    from paper_1511_03645_b200 import _lib, adjoint, device, solver
    nxa, nya = 16, 128
    shapes = [((0, 0), (20, 256)), ((20, 256), (18, 128)), ((40, 0), (8, 384))]
    _, patches = _level(shapes, seed=8)
    vals, wet, store = _store_n(9, nxa, nya, dry)
    t, window = 0.3, adjoint.TimeWindow(0.0, 0.75)
    tol = 0.7
    var = _lib.VARIANT_EXACT if variant == "exact" else _lib.VARIANT_FAST
    flags, counts, best = adjoint.flag_level(patches, t, store, window, tol, want_best=True, variant=var)
    st = solver.store_of(patches[0])
    tabs = device.flag_axis_tables(st, (nxa, nya), (0.0, 0.0), 1.0 / nxa, 1.0 / nya, (0.0, 0.0),
                                   patches[0].spec.dx, patches[0].spec.dy)
    assert tabs[5] is True
    idx = adjoint.query_window_times(t, window, _FakeStore(window))
    assert len(idx) >= 2
    for p, f, c, b in zip(patches, flags, counts, best):
        lo, shape, dx, dy = p.spec.lo, p.spec.shape, p.spec.dx, p.spec.dy
        x = (np.arange(lo[0], lo[0] + shape[0]) + 0.5) * dx
        y = (np.arange(lo[1], lo[1] + shape[1]) + 0.5) * dy
        xc, yc = np.broadcast_to(x[:, None], shape), np.broadcast_to(y[None, :], shape)
        ref = O.inner_product(p.state[:, 2:-2, 2:-2], xc, yc, vals, idx, (0.0, 0.0), 1.0 / nxa, 1.0 / nya,
                              p.aux.wet[2:-2, 2:-2], wet)
        if variant == "exact":
            assert np.array_equal(b, ref)
            assert np.array_equal(f, ref > tol)
        else:
            assert np.max(np.abs(b - ref)) <= 1e-12 * np.max(np.abs(ref))
            far = np.abs(ref - tol) > 1e-12 * tol
            assert np.array_equal(f[far], (ref > tol)[far])
        assert c == int(f.sum())


@pytest.mark.parametrize("case", ["span", "snapshot", "empty"])
@pytest.mark.parametrize("dry", [False, True])
def test_direct_kernel_equal_grids(dry, case):
    """Adjoint grid equal to the forward grid (64 x 512 under the 64 x 512
    level, as in C3): every interpolation weight is exactly 0 or 1, so
    windows of >= 2 snapshots run the direct kernel (k3_direct) -- bitwise
    equal to the reference arithmetic."""
    from paper_1511_03645_b200 import adjoint, device, solver
    nxa, nya = 64, 512
    _, patches = _level(ROWS, seed=11)
    vals, wet, store = _store_n(12, nxa, nya, dry)
    t, window = {"span": (0.3, adjoint.TimeWindow(0.0, 0.75)), "snapshot": (0.6, adjoint.TimeWindow(0.6, 0.6)),
                 "empty": (1.5, adjoint.TimeWindow(0.0, 1.0))}[case]   # empty: t past the last snapshot
    tol = 0.7 if case != "empty" else 0.0
    flags, counts, best = adjoint.flag_level(patches, t, store, window, tol, want_best=True)
    st = solver.store_of(patches[0])
    tabs = device.flag_axis_tables(st, (nxa, nya), (0.0, 0.0), 1.0 / nxa, 1.0 / nya, (0.0, 0.0),
                                   patches[0].spec.dx, patches[0].spec.dy)
    assert tabs[6] is True
    idx = adjoint.query_window_times(t, window, _FakeStore(window))
    assert len(idx) == {"span": len(idx) if len(idx) >= 2 else -1, "snapshot": 1, "empty": 0}[case]
    if case == "empty":   # the reference's inner product is zero everywhere (adjoint.py:227-249)
        assert not any(np.any(b) for b in best) and not any(f.any() for f in flags) and not any(counts)
        return
    for p, f, c, b in zip(patches, flags, counts, best):
        lo, shape, dx, dy = p.spec.lo, p.spec.shape, p.spec.dx, p.spec.dy
        x = (np.arange(lo[0], lo[0] + shape[0]) + 0.5) * dx
        y = (np.arange(lo[1], lo[1] + shape[1]) + 0.5) * dy
        xc, yc = np.broadcast_to(x[:, None], shape), np.broadcast_to(y[None, :], shape)
        ref = O.inner_product(p.state[:, 2:-2, 2:-2], xc, yc, vals, idx, (0.0, 0.0), 1.0 / nxa, 1.0 / nya,
                              p.aux.wet[2:-2, 2:-2], wet)
        assert np.array_equal(b, ref)
        assert np.array_equal(f, ref > tol)
        assert c == int(f.sum())


@pytest.mark.parametrize("variant", ["exact", "fast"])
@pytest.mark.parametrize("dry", [False, True])
@pytest.mark.parametrize("scale", [1e-3, 1.0])
def test_quad_window_pruning_keeps_flags(variant, dry, scale):
    """Flags-only calls on multi-snapshot windows prune cells whose envelope
    bound sum_c |q_c| max|qhat_c| cannot reach the tolerance
    (AdjFlagArgs.envelope).  Forward state: a localized bump (most cells far
    below the tolerance, some cells near it) -- flags and raw counts equal
    the reference's windowed max > tol (EXACT: the reference arithmetic;
    FAST: away from the tolerance) and the unpruned run's, bit for bit."""
    from paper_1511_03645_b200 import _lib, adjoint, device
    nxa, nya = 16, 128
    shapes = [((0, 0), (20, 256)), ((20, 256), (18, 128)), ((40, 0), (8, 384))]
    _, patches = _level(shapes, seed=8)
    for p in patches:      # a bump centred in the level: far cells are tiny
        cs = p.spec.cell_centers(include_ghost=True)
        X, Y = np.meshgrid(cs[0], cs[1], indexing="ij")
        env = scale * np.exp(-((X - 0.4) ** 2 + (Y - 0.5) ** 2) / 0.02)
        p.state = p.state * env[None]
    vals, wet, store = _store_n(9, nxa, nya, dry)
    t, window = 0.3, adjoint.TimeWindow(0.0, 0.75)
    var = _lib.VARIANT_EXACT if variant == "exact" else _lib.VARIANT_FAST
    idx = adjoint.query_window_times(t, window, _FakeStore(window))
    assert len(idx) >= 2
    refs = []
    for p in patches:
        lo, shape, dx, dy = p.spec.lo, p.spec.shape, p.spec.dx, p.spec.dy
        x = (np.arange(lo[0], lo[0] + shape[0]) + 0.5) * dx
        y = (np.arange(lo[1], lo[1] + shape[1]) + 0.5) * dy
        xc, yc = np.broadcast_to(x[:, None], shape), np.broadcast_to(y[None, :], shape)
        refs.append(O.inner_product(p.state[:, 2:-2, 2:-2], xc, yc, vals, idx, (0.0, 0.0), 1.0 / nxa, 1.0 / nya,
                                    p.aux.wet[2:-2, 2:-2], wet))
    tol = float(np.quantile(np.concatenate([r.ravel() for r in refs]), 0.97))   # ~3% flagged
    assert tol > 0
    old = device.USE_FLAG_PRUNING
    try:
        device.USE_FLAG_PRUNING = True
        fp, cp, _ = adjoint.flag_level(patches, t, store, window, tol, variant=var)
        device.USE_FLAG_PRUNING = False
        fu, cu, _ = adjoint.flag_level(patches, t, store, window, tol, variant=var)
    finally:
        device.USE_FLAG_PRUNING = old
    assert cp == cu
    for a, b, ref in zip(fp, fu, refs):
        assert np.array_equal(a, b)
        if variant == "exact":
            assert np.array_equal(a, ref > tol)
        else:
            far = np.abs(ref - tol) > 1e-12 * tol
            assert np.array_equal(a[far], (ref > tol)[far])
    assert sum(cp) > 0
