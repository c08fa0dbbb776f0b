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


@pytest.mark.parametrize("ni,nj", [(20, 16), (16, 17)])
def test_exact_oversized_tile_reported(ni, nj):
    """An ABI caller passing an EXACT tile larger than adj_step_tile_shape
    (16 x 16) gets nonfinite[patch] = 2 and an untouched output instead of a
    shared-memory overflow (the tiled kernel's face tables hold 16 x 16)."""
    import torch
    from paper_1511_03645_b200 import _lib, device, solver
    d = STEP[sorted(STEP)[0]]
    eq = make_equation(d["name"], gravity=d["gravity"] or 9.81)
    _, p = patch_from_arrays(d["q_in"], d["aux"], eq.is_swe, d["dx"], d["dy"], gravity=d["gravity"] or 9.81)
    st = solver.store_of(p)
    st.sync_in()
    out = st._free(st.cur)
    before = st.buf[out].clone()
    bad_tile = np.array([(0, 0, 0, ni, nj, 0)], dtype=_lib.TILE_DTYPE)
    st._tiles[_lib.VARIANT_EXACT] = (device._dev_table(bad_tile), 1, None, 1)
    _, nf = device.launch_step(st, d["dt"], eq, d["limiter"], _lib.VARIANT_EXACT, out)
    torch.cuda.synchronize()
    assert int(nf[0].item()) == 2
    assert torch.equal(st.buf[out], before)
    del st._tiles[_lib.VARIANT_EXACT]


def test_packed_jobs_need_static_speed():
    """FAST with a job table but no static CFL bound is rejected (ADJ_ERR_BAD_ARG)
    instead of launching nothing."""
    from paper_1511_03645_b200 import _lib
    a = _lib.AdjStepArgs()
    a.ntile, a.njob, a.ndim, a.variant, a.system = 1, 1, 2, _lib.VARIANT_FAST, 1
    a.ghost, a.dt, a.limiter = 2, 1.0, _lib.LIMITERS["MC"]
    # any non-null pointers: the call is rejected before a launch reads them
    a.q_in, a.q_out, a.aux, a.patches, a.tiles, a.speed_max, a.nonfinite, a.work_counter = range(8, 72, 8)
    a.job_offsets = 80
    a.static_speed = 0
    assert _lib.lib().adj_step_level(_lib.C.byref(a)) == 5
