"""The CUDA-graph replay of the level sweep reproduces the eager sweep
bitwise (states, times, counters)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def small_hierarchy(variant):
    from paper_1511_03645_b200 import amr, solver
    from paper_1511_03645_b200 import equations as E
    from paper_1511_03645_b200.geometry import PatchHierarchy
    eq = E.Acoustics2D(E.AcousticsMaterialModel(
        lambda x, y: np.where(np.asarray(y) < 0.2 * np.asarray(x) + 0.3, 4.0, 1.0),
        lambda x, y: np.ones_like(np.asarray(x, float))))
    ctx = amr.AmrContext(equation=eq, boundary=solver.BoundarySpec("wall", "outflow", "outflow", "wall"),
                         strategy=amr.EverywhereFlagging(), regrid_interval=10 ** 9, variant=variant)
    h = PatchHierarchy(xlim=(0.0, 1.0), ylim=(0.0, 1.0), base_shape=(64, 64), ratios=[2, 4])
    boxes = [
        [((i * 16, j * 16), (i * 16 + 15, j * 16 + 15)) for i in range(4) for j in range(4)],
        [((32, 32), (63, 63)), ((64, 32), (95, 63)), ((32, 64), (63, 95)), ((16, 96), (47, 111))],
        [((160, 160), (191, 191)), ((192, 160), (223, 191)), ((160, 224), (191, 255))],
    ]
    h.levels = []
    for lev, bl in enumerate(boxes, start=1):
        ps = []
        for lo, hi in bl:
            p = amr.make_patch(h, lev, lo, hi, ctx, time=0.0)
            cs = p.spec.cell_centers()
            X, Y = np.meshgrid(cs[0], cs[1], indexing="ij")
            p.interior()[0] = np.exp(-60.0 * ((X - 0.45) ** 2 + (Y - 0.55) ** 2))
            ps.append(p)
        h.levels.append(ps)
    return h, ctx, solver.select_dt(h, eq, 0.9)


def test_sweep_graph_matches_eager():
    from paper_1511_03645_b200 import _lib, amr
    ha, ca, dt = small_hierarchy(_lib.VARIANT_FAST)
    hb, cb, _ = small_hierarchy(_lib.VARIANT_FAST)
    for _ in range(8):
        amr.advance_hierarchy(ha, 1, dt, ca)
    g = amr.SweepGraph(hb, dt, cb)          # 2 eager warm-up + 2 captured steps
    g.advance(4)
    assert ca.cell_steps == cb.cell_steps and ca.step_counts == cb.step_counts
    for lev in (1, 2, 3):
        for pa, pb in zip(ha.patches(lev), hb.patches(lev)):
            assert pa.time == pb.time
            assert np.array_equal(pa.interior(), pb.interior())


def test_sweep_graph_lite_shadow_matches_eager():
    """After its first pair (full shadow + lite shadow, compared), replays use
    the lite host bookkeeping; many pairs later the states, times and
    counters still equal the eager sweep bitwise."""
    from paper_1511_03645_b200 import _lib, amr
    ha, ca, dt = small_hierarchy(_lib.VARIANT_FAST)
    hb, cb, _ = small_hierarchy(_lib.VARIANT_FAST)
    for _ in range(4 + 14):
        amr.advance_hierarchy(ha, 1, dt, ca)
    g = amr.SweepGraph(hb, dt, cb)
    g.advance(2)
    assert g.lite_ok is True
    g.advance(12)
    assert ca.cell_steps == cb.cell_steps and ca.step_counts == cb.step_counts
    for lev in (1, 2, 3):
        for pa, pb in zip(ha.patches(lev), hb.patches(lev)):
            assert pa.time == pb.time and pa.time_old == pb.time_old
            assert np.array_equal(pa.interior(), pb.interior())


def test_sweep_graph_overlap_used():
    """The captured sweep overlaps parent steps with the first substep of the
    finer level (side streams); with the FAST weight snap every replayed
    pair may use it."""
    from paper_1511_03645_b200 import _lib, amr
    if not amr.USE_LEVEL_OVERLAP:
        pytest.skip("level overlap disabled (ADJAMR_LEVEL_OVERLAP=0)")
    hb, cb, dt = small_hierarchy(_lib.VARIANT_FAST)
    g = amr.SweepGraph(hb, dt, cb)
    g.advance(8)
    assert g.skip_slots and g.graph_seq is not None
    assert g.seq_replays == 0


def test_sweep_graph_sequential_fallback(monkeypatch):
    """Without the weight snap, first-substep weights pick up the level
    clocks' rounding drift; pairs with such a weight replay the sequential
    capture, and the result still equals the eager sweep bitwise."""
    from paper_1511_03645_b200 import _lib, amr
    monkeypatch.setattr(amr, "SNAP_W", 0.0)
    ha, ca, dt = small_hierarchy(_lib.VARIANT_FAST)
    hb, cb, _ = small_hierarchy(_lib.VARIANT_FAST)
    for _ in range(4 + 20):
        amr.advance_hierarchy(ha, 1, dt, ca)
    g = amr.SweepGraph(hb, dt, cb)
    g.advance(20)
    assert ca.cell_steps == cb.cell_steps and ca.step_counts == cb.step_counts
    for lev in (1, 2, 3):
        for pa, pb in zip(ha.patches(lev), hb.patches(lev)):
            assert pa.time == pb.time and pa.time_old == pb.time_old
            assert np.array_equal(pa.interior(), pb.interior())
