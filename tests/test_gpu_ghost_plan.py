"""The planned level fill (one gather launch: coarse interpolation, same-level
copies and physical boundaries compiled per regrid, adj_ghost_plan_build /
adj_fill_ghost_plan) writes exactly the values of the three-phase fill
(fill_level_ghosts, amr.py:479-491) -- compared bitwise on whole
ghost-inclusive level buffers, at a mid-interval coarse time weight."""
import numpy as np
import pytest

from tests.amr_cases import CASES
from tests.test_gpu_amr import setup

pytestmark = pytest.mark.gpu


def _fill_all(h, ctx, plan):
    from paper_1511_03645_b200 import amr
    old = amr.USE_GHOST_PLAN
    amr.USE_GHOST_PLAN = plan
    out = []
    try:
        for lev in range(1, h.num_levels() + 1):
            ps = h.patches(lev)
            if not ps:
                continue
            st = amr._plan(h, lev).st
            t = ps[0].time
            if lev >= 2:
                cp = h.patches(lev - 1)[0]
                if cp.time_old is not None and cp.time_old < cp.time:
                    t = 0.5 * (cp.time_old + cp.time)       # blend old/new coarse states
            amr.fill_level_ghosts(h, lev, t, ctx)
            out.append(st.buf[st.cur].clone())
    finally:
        amr.USE_GHOST_PLAN = old
    return out


@pytest.mark.parametrize("name", sorted(CASES))
def test_planned_fill_equals_three_phase_fill(name):
    import torch
    from paper_1511_03645_b200 import _lib, amr
    h, ctx, dt, case = setup(name, _lib.VARIANT_EXACT)
    amr.advance_hierarchy(h, 1, dt, ctx)
    # coarse levels carry a saved state from the last step: fills interpolate in time
    ref = _fill_all(h, ctx, plan=False)
    got = _fill_all(h, ctx, plan=True)
    torch.cuda.synchronize()
    assert len(ref) == len(got) and ref
    for lev, (a, b) in enumerate(zip(ref, got), start=1):
        assert torch.equal(a, b), (name, lev, int((a != b).sum()))
    # the planned path was used on every level
    for lev in range(1, h.num_levels() + 1):
        if h.patches(lev):
            assert amr._plan(h, lev)._gather, lev


def test_plan_counts_physical_cells():
    from paper_1511_03645_b200 import _lib, amr, device
    h, ctx, dt, case = setup("ac2d_adjoint", _lib.VARIANT_EXACT)
    amr.fill_level_ghosts(h, 1, 0.0, ctx)
    gp = next(iter(amr._plan(h, 1)._gather.values()))
    st = amr._plan(h, 1).st
    assert gp.n == gp.nc + int((amr._plan(h, 1).copies.np["ni"] * amr._plan(h, 1).copies.np["nj"]).sum()) + \
        device.physical_cell_count(st, h.level_shape(1))
    assert np.isfinite(gp.n)


@pytest.mark.parametrize("name", sorted(CASES))
def test_planned_restrict_equals_rect_restrict(name):
    import torch
    from paper_1511_03645_b200 import _lib, amr
    h, ctx, dt, case = setup(name, _lib.VARIANT_EXACT)
    amr.advance_hierarchy(h, 1, dt, ctx)
    done = 0
    for lev in range(h.num_levels() - 1, 0, -1):
        if not h.patches(lev + 1):
            continue
        fpl = amr._plan(h, lev + 1)
        outs = []
        for plan in (False, True):
            amr.USE_RESTRICT_PLAN = plan
            fpl.restrict_to = None
            try:
                before = fpl.cst.buf[fpl.cst.cur].clone()
                amr.restrict_fine_to_coarse(h, lev)
                outs.append(fpl.cst.buf[fpl.cst.cur].clone())
                fpl.cst.buf[fpl.cst.cur].copy_(before)
            finally:
                amr.USE_RESTRICT_PLAN = True
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1]), (name, lev, int((outs[0] != outs[1]).sum()))
        done += 1
    assert done


@pytest.mark.parametrize("name", ["ac2d_adjoint", "ac2d_hetero", "ac2d_everywhere"])
def test_fused_fill_equals_separate_fill(name):
    """The planned fill run inside the step launch (prefill + grid barrier)
    gives bitwise the states of the separate gather launch (FAST variant,
    several coarse steps incl. regrids).  The fused restriction is off in
    both runs (a prefilled step never fuses it; its block sums would differ
    in the last bit)."""
    from paper_1511_03645_b200 import _lib, amr
    from tests.test_gpu_amr import run
    outs = []
    for fused in (False, True):
        old, old_r = amr.USE_FUSED_FILL, amr.USE_FUSED_RESTRICT
        amr.USE_FUSED_FILL = fused
        amr.USE_FUSED_RESTRICT = False
        try:
            outs.append(run(name, _lib.VARIANT_FAST))
        finally:
            amr.USE_FUSED_FILL, amr.USE_FUSED_RESTRICT = old, old_r
    for step, (a, b) in enumerate(zip(*outs)):
        assert a["nlev"] == b["nlev"] and a["flagged"] == b["flagged"]
        for lev in range(1, a["nlev"] + 1):
            assert np.array_equal(a[f"L{lev}_boxes"], b[f"L{lev}_boxes"])
            assert np.array_equal(a[f"L{lev}_q"], b[f"L{lev}_q"]), (name, step, lev)
