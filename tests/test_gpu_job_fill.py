"""Level ghost fill fused into the step launch per warp job (AdjJobFill,
amr.USE_JOB_FILL, opt-in): the FAST AMR runs with the per-job fill equal
the runs with the separate planned gather launch bitwise (same entries, same
arithmetic, same step), the cached coarse values of an interval's later
substeps included -- so the reference parity of test_gpu_amr's FAST runs
(separate gather) carries over."""
import numpy as np
import pytest

from tests.amr_cases import CASES
from tests.test_gpu_amr import run

pytestmark = pytest.mark.gpu

TWO_D = [n for n in sorted(CASES) if CASES[n]["ndim"] == 2]


def _spy(modes):
    from paper_1511_03645_b200 import device
    orig = device.launch_step

    def spy(*a, **k):
        jf = k.get("job_fill")
        if jf is not None:
            modes.append(int(jf.cache_mode) if jf.c_base else -1)
        return orig(*a, **k)
    return orig, spy


def _run(name, on):
    from paper_1511_03645_b200 import _lib, amr, device
    old = amr.USE_JOB_FILL
    amr.USE_JOB_FILL = on
    modes = []
    orig, spy = _spy(modes)
    device.launch_step = spy
    try:
        return run(name, _lib.VARIANT_FAST), modes
    finally:
        amr.USE_JOB_FILL = old
        device.launch_step = orig


@pytest.mark.parametrize("name", TWO_D)
def test_job_fill_matches_separate_gather(name):
    on, modes = _run(name, True)
    off, none = _run(name, False)
    assert not none
    for a, b in zip(on, off):
        assert a["nlev"] == b["nlev"] and a["flagged"] == b["flagged"] and a["cell_steps"] == b["cell_steps"]
        for lev in range(1, a["nlev"] + 1):
            assert np.array_equal(a[f"L{lev}_boxes"], b[f"L{lev}_boxes"])
            assert np.array_equal(a[f"L{lev}_q"], b[f"L{lev}_q"])
    if name != "swe_basin":          # the dry shore runs the EXACT step (no job fill)
        assert modes, "the job-fill path was not taken"


def _c5_levels(h):
    return [np.concatenate([p.state.reshape(3, -1) for p in h.patches(lev)], axis=1) for lev in (1, 2, 3)]


@pytest.mark.parametrize("graph", [False, True])
def test_c5_job_fill_equals_gather(graph):
    """C5-like hierarchy (32^2 patches, ratios 2 and 4): two coarse steps with
    the per-job fill (eager, or replayed from the captured sweep graph) equal
    the separate-gather run bitwise on every ghost-inclusive patch box; the
    L2 and L3 fills compute their coarse values in an interval's first
    substep (cache mode 1) and reuse them after (mode 2)."""
    import bench
    from paper_1511_03645_b200 import _lib, amr, device
    res = {}
    for on in (True, False):
        amr.USE_JOB_FILL = on
        modes = []
        orig, spy = _spy(modes)
        device.launch_step = spy
        try:
            h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
            if graph and on:
                g = amr.SweepGraph(h, dt, ctx)     # two warm-up coarse steps, two captured (replayed once)
                g.advance(2)
            else:
                for _ in range(6 if graph else 2):
                    amr.advance_hierarchy(h, 1, dt, ctx)
            res[on] = (_c5_levels(h), list(modes))
        finally:
            amr.USE_JOB_FILL = False
            device.launch_step = orig
    for a, b in zip(res[True][0], res[False][0]):
        assert np.array_equal(a, b)
    modes = res[True][1]
    assert -1 in modes and 1 in modes and 2 in modes     # L1 (no coarse), first and later substeps
    assert not res[False][1]


def test_job_fill_abi_validation():
    """A job fill without job_offsets, or a cache mode without a cache, is rejected."""
    from paper_1511_03645_b200 import _lib
    a = _lib.AdjStepArgs()
    a.ntile, a.njob, a.ndim, a.variant, a.system = 1, 1, 2, _lib.VARIANT_FAST, 1
    a.ghost, a.dt, a.limiter = 2, 1.0, _lib.LIMITERS["MC"]
    a.q_in, a.q_out, a.aux, a.patches, a.tiles, a.speed_max, a.nonfinite, a.work_counter = range(8, 72, 8)
    a.static_speed = 80
    a.flags = _lib.STEP_COUNTER_ZERO
    a.job_fill.n = 10
    a.job_fill.entry_off, a.job_fill.dst, a.job_fill.src, a.job_fill.meta = 88, 96, 104, 112
    assert _lib.lib().adj_step_level(_lib.C.byref(a)) == 5          # no job_offsets
    a.job_offsets = 120
    a.job_fill.cache_mode = 1
    assert _lib.lib().adj_step_level(_lib.C.byref(a)) == 5          # cache mode without a cache
