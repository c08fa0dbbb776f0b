"""K1 parity on the GPU against the reference's golden vectors."""
import numpy as np
import pytest

from tests.golden_io import load
from tests.helpers import make_equation, norm_rel, patch_from_arrays

STEP = load("step.npz")
pytestmark = pytest.mark.gpu


def _run(d, variant):
    from paper_1511_03645_b200 import solver
    eq = make_equation(d["name"], gravity=d["gravity"] or 9.81)
    _, p = patch_from_arrays(d["q_in"], d["aux"], eq.is_swe, d["dx"], d["dy"], gravity=d["gravity"] or 9.81)
    res = solver.step_patch(p, d["dt"], eq, d["limiter"], variant=variant)
    return p.state.copy(), res.max_courant


@pytest.mark.parametrize("case", sorted(STEP))
def test_exact_variant_bitwise(case):
    from paper_1511_03645_b200 import _lib
    d = STEP[case]
    q, cfl = _run(d, _lib.VARIANT_EXACT)
    assert np.array_equal(q, d["q_out"]), norm_rel(q, d["q_out"])
    assert cfl == d["cfl"]


@pytest.mark.parametrize("case", sorted(STEP))
def test_fast_variant_1e12(case):
    from paper_1511_03645_b200 import _lib
    d = STEP[case]
    q, cfl = _run(d, _lib.VARIANT_FAST)
    # tolerance stated by BASELINE.json north_star: 1e-12 relative (fp64), norm-relative per component
    assert norm_rel(q, d["q_out"]) <= 1e-12
    assert abs(cfl - d["cfl"]) <= 1e-14 * max(1.0, d["cfl"])
    # ghosts are untouched by a step (solver.py:508 updates the interior only)
    g = 2
    mask = np.ones(q.shape[1:], bool)
    mask[(slice(g, -g),) * (q.ndim - 1)] = False
    assert np.array_equal(q[:, mask], d["q_out"][:, mask])


def test_cfl_violation_raises_before_mutation():
    from paper_1511_03645_b200 import solver
    d = STEP["step00"]
    eq = make_equation(d["name"])
    _, p = patch_from_arrays(d["q_in"], d["aux"], False, d["dx"], d["dy"])
    with pytest.raises(solver.CflViolationError):
        solver.step_patch(p, d["dt"] * 2.0, eq, "MC")
    assert np.array_equal(p.state, d["q_in"])
    assert p.time == 0.0


def test_nonfinite_raises():
    from paper_1511_03645_b200 import solver
    d = STEP["step00"]
    eq = make_equation(d["name"])
    q = d["q_in"].copy()
    q[0, 5, 5] = np.nan
    _, p = patch_from_arrays(q, d["aux"], False, d["dx"], d["dy"])
    with pytest.raises(solver.NumericalBlowupError):
        solver.step_patch(p, d["dt"], eq, "MC")


def test_bad_args():
    from paper_1511_03645_b200 import solver
    d = STEP["step00"]
    eq = make_equation(d["name"])
    _, p = patch_from_arrays(d["q_in"], d["aux"], False, d["dx"], d["dy"])
    with pytest.raises(ValueError):
        solver.step_patch(p, 0.0, eq)
    with pytest.raises(ValueError):
        solver.step_patch(p, d["dt"], eq, "vanleer")


@pytest.mark.parametrize("rows", ["1", "2"])
@pytest.mark.parametrize("case", [c for c in sorted(STEP) if not STEP[c]["name"].startswith("ac1d")
                                  and STEP[c]["name"] != "swe_dry" and STEP[c]["name"] != "swe_adj_rev"])
def test_fast_kernel_rows_per_lane(case, rows, monkeypatch):
    """Both fast kernels (one and two rows per lane) on every golden 2D case
    without dry cells, forced through ADJAMR_K1_ROWS."""
    from paper_1511_03645_b200 import _lib
    monkeypatch.setenv("ADJAMR_K1_ROWS", rows)
    d = STEP[case]
    q, cfl = _run(d, _lib.VARIANT_FAST)
    assert norm_rel(q, d["q_out"]) <= 1e-12
