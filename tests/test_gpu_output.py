"""Output path on the device against the reference's own
values (tests/golden/output.npz): evaluate_J within 1e-12 of sum |terms|
(per-cell products are the reference's; only the summation order differs),
gauges bitwise, snapshot records equal to the patch interiors."""
import numpy as np
import pytest

from oracle import adjamr_oracle as O
from tests.golden_io import load
from tests.test_gpu_amr import setup
from tests.test_oracle_output import golden_levels

pytestmark = pytest.mark.gpu
OUT = load("output.npz")
AMR = load("amr.npz")


def _hier(name):
    from paper_1511_03645_b200 import _lib, amr
    h, ctx, dt, case = setup(name, _lib.VARIANT_EXACT)
    amr.advance_hierarchy(h, 1, dt, ctx)      # == the golden state after coarse step 0
    return h, ctx


def _scale(name, qh):
    """sum over uncovered cells of |qhat . q| * area (conditioning of J)."""
    levels, ratios, origin, widths, shapes, a_dx, a_dy = golden_levels(name)
    absl = [[(lo, np.abs(q)) for lo, q in lev] for lev in levels]
    return O.evaluate_J(absl, ratios, origin, widths, np.abs(qh), origin, a_dx, a_dy)


@pytest.mark.parametrize("name", sorted(OUT))
def test_evaluate_J_matches_reference(name):
    from paper_1511_03645_b200 import output
    h, ctx = _hier(name)
    store = ctx.strategy.store
    g, o = AMR[name], OUT[name]
    for t, want in zip(o["J_times"], o["J_store"]):
        got = output.evaluate_J(h, store, float(t))
        scale = _scale(name, O.interpolate_time(g["store_fields"], g["store_times"], float(t)))
        assert abs(got - want) <= 1e-12 * scale, (t, got, want, scale)
    got = output.evaluate_J(h, store.fields[-1], 0.0)
    assert abs(got - o["J_phi"][0]) <= 1e-12 * _scale(name, g["store_fields"][-1])


@pytest.mark.parametrize("name", sorted(OUT))
def test_gauges_match_reference_bitwise(name):
    from paper_1511_03645_b200 import output
    h, ctx = _hier(name)
    o = OUT[name]
    series = [output.GaugeSeries(k, tuple(float(v) for v in loc)) for k, loc in enumerate(o["gauge_locs"])]
    output.record_gauges(h, series, float(o["t"]))
    for s, want, found in zip(series, o["gauge_vals"], o["gauge_found"]):
        assert bool(s.values) == bool(found)
        if s.values:
            assert s.times == [float(o["t"])]
            assert np.array_equal(s.values[0], want), (s.location, s.values[0], want)


@pytest.mark.parametrize("name", sorted(OUT))
def test_snapshot_records_are_the_interiors(name, tmp_path):
    from paper_1511_03645_b200 import output
    h, ctx = _hier(name)
    recs = output.snapshot_records(h)
    want = []
    for lev in range(1, h.num_levels() + 1):
        for p in sorted(h.patches(lev), key=lambda q: q.spec.lo):
            want.append((lev, p.spec.lo, np.array(p.interior())))
    assert [(r.level, r.lo) for r in recs] == [(w[0], w[1]) for w in want]
    for r, w in zip(recs, want):
        assert np.array_equal(r.values, w[2])
    path = tmp_path / "snap.txt"
    output.write_snapshot(h, str(path))
    first = path.read_text().splitlines()[0]
    assert first.startswith("patch level=1 lo=")


def test_evaluate_J_uniform_field_source():
    """UniformField source (adjoint.py:313-321): device vs the oracle's
    per-cell products summed in numpy order, within 1e-12 of sum |terms|."""
    from paper_1511_03645_b200 import output
    from paper_1511_03645_b200.geometry import UniformField
    rng = np.random.default_rng(5)
    src = UniformField(values=rng.standard_normal((3, 40, 30)), origin=(-1.0, 0.5), dx=0.05, dy=0.04, time=0.0)
    phi = UniformField(values=rng.standard_normal((3, 25, 20)), origin=(-1.0, 0.5), dx=0.08, dy=0.06, time=0.0)
    got = output.evaluate_J(src, phi, 0.0)
    cs = src.centers()
    x = np.broadcast_to(cs[0][:, None], (40, 30))
    y = np.broadcast_to(cs[1][None, :], (40, 30))
    qh = O.uniform_sample(phi.values, phi.origin, phi.dx, phi.dy, x, y)
    want = float(np.sum(qh * src.values) * src.dx * src.dy)
    scale = float(np.sum(np.abs(qh * src.values)) * src.dx * src.dy)
    assert abs(got - want) <= 1e-12 * scale
