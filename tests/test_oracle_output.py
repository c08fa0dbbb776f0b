"""Oracle restatement of the output path (evaluate_J, gauges) pinned to the
reference's own values (tests/golden/make_golden_output.py) -- bitwise."""
import numpy as np
import pytest

from oracle import adjamr_oracle as O
from tests.amr_cases import CASES
from tests.golden_io import load

AMR = load("amr.npz")
OUT = load("output.npz")
NAMES = sorted(OUT)


def golden_levels(name):
    """Levels after coarse step 0 as [(lo, interior q)], plus geometry."""
    case, g = CASES[name], AMR[name]
    nd = case["ndim"]
    levels = []
    for lev in range(1, int(g["s0_nlev"]) + 1):
        boxes, q = g[f"s0_L{lev}_boxes"], g[f"s0_L{lev}_q"]
        ps, off = [], 0
        for b in boxes:
            lo, hi = tuple(int(v) for v in b[:nd]), tuple(int(v) for v in b[nd:])
            shape = tuple(h - l + 1 for l, h in zip(lo, hi))
            n = int(np.prod(shape))
            ps.append((lo, q[:, off:off + n].reshape(q.shape[0], *shape)))
            off += n
        levels.append(ps)
    ratios = list(case["ratios"])
    origin = (case["xlim"][0],) if nd == 1 else (case["xlim"][0], case["ylim"][0])
    widths, shapes, cum = [], [], 1
    for li in range(len(levels)):
        if li:
            cum *= ratios[li - 1]
        wx = (case["xlim"][1] - case["xlim"][0]) / (case["base"][0] * cum)
        wy = 0.0 if nd == 1 else (case["ylim"][1] - case["ylim"][0]) / (case["base"][1] * cum)
        widths.append((wx, wy))
        shapes.append(tuple(n * cum for n in case["base"]))
    shp = case["adjoint_shape"]
    a_dx = (case["xlim"][1] - case["xlim"][0]) / shp[0]
    a_dy = 0.0 if nd == 1 else (case["ylim"][1] - case["ylim"][0]) / shp[1]
    return levels, ratios, origin, widths, shapes, a_dx, a_dy


@pytest.mark.parametrize("name", NAMES)
def test_oracle_evaluate_J_matches_reference(name):
    levels, ratios, origin, widths, shapes, a_dx, a_dy = golden_levels(name)
    g, o = AMR[name], OUT[name]
    fields, times = g["store_fields"], g["store_times"]
    for t, want in zip(o["J_times"], o["J_store"]):
        qh = O.interpolate_time(fields, times, float(t))
        assert O.evaluate_J(levels, ratios, origin, widths, qh, origin, a_dx, a_dy) == want
    assert O.evaluate_J(levels, ratios, origin, widths, fields[-1], origin, a_dx, a_dy) == o["J_phi"][0]


@pytest.mark.parametrize("name", NAMES)
def test_oracle_gauges_match_reference(name):
    levels, ratios, origin, widths, shapes, a_dx, a_dy = golden_levels(name)
    o = OUT[name]
    for loc, want, found in zip(o["gauge_locs"], o["gauge_vals"], o["gauge_found"]):
        hit = O.finest_patch_at(levels, origin, widths, shapes, tuple(loc))
        assert (hit is not None) == bool(found)
        if hit is None:
            continue
        lo, q = levels[hit[0]][hit[1]]
        got = O.gauge_value(q, lo, origin, widths[hit[0]], tuple(loc))
        assert np.array_equal(got, want)
