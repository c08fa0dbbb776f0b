"""K5 (adj_flag_level_mask): the device post-processing of adjoint flags --
region overrides, clipped box buffering, level-mask OR, proper-nesting clip --
equals the host path (flag_cells / buffer_flags / allowed_region_mask,
amr.py:137-179, 570-581, geometry.py:341-368) cell for cell, with the same
raw count."""
import numpy as np
import pytest

from tests.test_gpu_amr import setup

pytestmark = pytest.mark.gpu


def _host(h, parent, parents, ctx):
    from paper_1511_03645_b200 import amr
    from paper_1511_03645_b200.geometry import allowed_region_mask
    mask = np.zeros(h.level_shape(parent), dtype=bool)
    raw = 0
    for ff in amr._flag_level(parents, ctx):
        raw += int(ff.flags.sum())
        bf = amr.buffer_flags(ff, ctx.buffer_cells)
        sl = amr._box_slice(ff.lo, tuple(l + n - 1 for l, n in zip(ff.lo, bf.flags.shape)))
        mask[sl] |= bf.flags
    allowed = allowed_region_mask(h, parent)
    return mask & allowed, allowed, raw


def _regions(case, nd):
    from paper_1511_03645_b200 import amr
    x0, x1 = case["xlim"]
    xs = (x0 + 0.3 * (x1 - x0), x0 + 0.55 * (x1 - x0))
    if nd == 1:
        return (amr.RefinementRegion(1, 4, 0.0, 1e9, xs),
                amr.RefinementRegion(1, 1, 0.0, 1e9, (x0 + 0.7 * (x1 - x0), x1)))
    y0, y1 = case["ylim"]
    return (amr.RefinementRegion(3, 4, 0.0, 1e9, (*xs, y0 + 0.2 * (y1 - y0), y0 + 0.45 * (y1 - y0))),     # force
            amr.RefinementRegion(1, 1, 0.0, 1e9, (x0 + 0.6 * (x1 - x0), x1, y0, y0 + 0.5 * (y1 - y0))),  # clear
            amr.RefinementRegion(1, 4, 5e8, 1e9, (x0, x1, y0, y1)))                                     # inactive


@pytest.mark.parametrize("name", ["ac2d_adjoint", "ac2d_hetero", "ac1d_adjoint"])
@pytest.mark.parametrize("regions", [False, True])
@pytest.mark.parametrize("buffer", [0, 1, 3])
def test_device_flag_mask_equals_host(name, regions, buffer):
    from paper_1511_03645_b200 import _lib, amr
    h, ctx, dt, case = setup(name, _lib.VARIANT_EXACT)
    amr.advance_hierarchy(h, 1, dt, ctx)
    ctx.buffer_cells = buffer
    if regions:
        ctx.regions = _regions(case, h.ndim)
    checked = 0
    for parent in range(1, h.num_levels() + 1):
        parents = h.patches(parent)
        if not parents:
            continue
        amr.fill_level_ghosts(h, parent, parents[0].time, ctx)
        got = amr._device_level_mask(h, parent, parents, parents[0].time, ctx)
        assert got is not None
        want = _host(h, parent, parents, ctx)
        assert np.array_equal(got[1], want[1]), (parent, "allowed")
        assert np.array_equal(got[0], want[0]), (parent, int((got[0] != want[0]).sum()))
        assert got[2] == want[2]
        checked += 1
    assert checked
