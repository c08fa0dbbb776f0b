"""Restriction fused into the finest level's last substep (AdjStepRestrict,
amr.USE_FUSED_RESTRICT): the FAST AMR runs with and without it agree to the
FAST tolerance (1e-12 norm-relative; only the block sum order differs), with
identical grids, flag counts and cell-step accounting; and the fused path
is taken.  The reference parity of the fused runs is test_gpu_amr's FAST
test (fusion is on by default)."""
import numpy as np
import pytest

from tests.amr_cases import CASES
from tests.helpers import norm_rel
from tests.test_gpu_amr import run

pytestmark = pytest.mark.gpu

TWO_D = [n for n in sorted(CASES) if CASES[n]["ndim"] == 2]


def _run(name, fused):
    from paper_1511_03645_b200 import _lib, amr
    old = amr.USE_FUSED_RESTRICT
    amr.USE_FUSED_RESTRICT = fused
    calls = []
    orig = amr.step_level

    def spy(*a, **k):
        did = orig(*a, **k)
        calls.append(did)
        return did
    amr.step_level = spy
    try:
        return run(name, _lib.VARIANT_FAST), sum(calls)
    finally:
        amr.USE_FUSED_RESTRICT = old
        amr.step_level = orig


@pytest.mark.parametrize("name", TWO_D)
def test_fused_restriction_matches_separate(name):
    fused, nf = _run(name, True)
    sep, ns = _run(name, False)
    assert ns == 0
    for a, b in zip(fused, sep):
        assert a["nlev"] == b["nlev"] and a["flagged"] == b["flagged"] and a["cell_steps"] == b["cell_steps"]
        for lev in range(1, a["nlev"] + 1):
            assert np.array_equal(a[f"L{lev}_boxes"], b[f"L{lev}_boxes"])
            assert norm_rel(a[f"L{lev}_q"], b[f"L{lev}_q"]) <= 1e-12
    if name in ("ac2d_adjoint", "ac2d_everywhere"):
        assert nf > 0, "the fused path was not taken"


def test_c5_sweep_fuses_finest_restriction():
    """C5-like hierarchy (32^2 patches, ratios 2 and 4): the L3 -> L2
    restriction is fused (two per coarse step), L2 -> L1 is not (L2 has
    children), and one coarse step matches the unfused step."""
    import bench
    from paper_1511_03645_b200 import _lib, amr
    res = {}
    for fused in (True, False):
        amr.USE_FUSED_RESTRICT = fused
        try:
            h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
            amr.advance_hierarchy(h, 1, dt, ctx)
            res[fused] = ([np.concatenate([p.interior().reshape(3, -1) for p in h.patches(lev)], axis=1)
                           for lev in (1, 2, 3)], ctx.__dict__.get("fused_restrictions", 0))
        finally:
            amr.USE_FUSED_RESTRICT = True
    assert res[True][1] == 2 and res[False][1] == 0
    for a, b in zip(res[True][0], res[False][0]):
        assert norm_rel(a, b) <= 1e-12
