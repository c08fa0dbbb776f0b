"""K3 parity on the GPU against the reference's golden vectors (bitwise)."""
import numpy as np
import pytest

from tests.golden_io import load
from tests.helpers import material_from_planes

FLAG = load("flag.npz")
pytestmark = pytest.mark.gpu


def _setup(d, nd=2):
    from paper_1511_03645_b200 import adjoint
    from paper_1511_03645_b200.geometry import Patch, PatchHierarchy, UniformField
    lo, shape = tuple(int(v) for v in d["lo"]), tuple(int(v) for v in d["shape"])
    if nd == 2:
        h = PatchHierarchy(xlim=(0.0, 1.2), ylim=(0.0, 1.0), base_shape=(48, 40), ratios=[])
    else:
        h = PatchHierarchy(xlim=(0.0, 2.0), ylim=None, base_shape=(80,), ratios=[])
    spec = h.make_spec(1, lo, tuple(l + n - 1 for l, n in zip(lo, shape)))
    assert spec.dx == d["dx"]
    p = Patch(spec, d["q"].shape[0])
    swe = nd == 2 and str(d["name"]).startswith("swe")
    if nd == 2:
        p.aux = material_from_planes(d["aux"], swe)
    else:
        from paper_1511_03645_b200 import equations as E
        one = np.ones(d["q"].shape[1])
        p.aux = E.AcousticsMaterial(bulk=one, rho=one, c=one, z=one)
    p.state = d["q"]
    origin = (0.0, 0.0) if nd == 2 else (0.0,)
    fields = [UniformField(values=d["fields"][k], origin=origin, dx=d["a_dx"], dy=d.get("a_dy", 0.0), time=t)
              for k, t in enumerate(d["times"])]
    window = adjoint.TimeWindow(1.0, 2.0) if nd == 2 else adjoint.TimeWindow(0.5, 1.0)
    wet = d["adj_wet"] if nd == 2 and d["adj_wet"].size else None
    store = adjoint.AdjointSnapshotStore(times=d["times"], fields=fields, window=window, wet=wet)
    return p, store


@pytest.mark.parametrize("case", ["flag0", "flag1", "flag2"])
def test_flags_and_values_bitwise(case):
    from paper_1511_03645_b200 import adjoint
    d = FLAG[case]
    p, store = _setup(d)
    for n, t in enumerate(d["t_list"]):
        assert adjoint.query_window_times(t, store.window, store) == list(d[f"idx{n}"])
        best = adjoint.inner_product_field(p, t, store, store.window)
        assert np.array_equal(best, d[f"best{n}"])
        ff = adjoint.inner_product_flags(p, t, store, store.window, d["tol"])
        assert np.array_equal(ff.flags, d[f"flags{n}"])
        _, counts, _ = adjoint.flag_level([p], t, store, store.window, d["tol"])
        assert counts[0] == int(d[f"flags{n}"].sum())


def test_flags_1d_bitwise():
    from paper_1511_03645_b200 import adjoint
    d = FLAG["flag1d"]
    p, store = _setup(d, nd=1)
    best = adjoint.inner_product_field(p, 0.3, store, store.window)
    assert np.array_equal(best, d["best"])


def test_time_interpolated_mode_matches_interpolate_time():
    """Mode 1 at a single instant equals |interpolate_time(t) . q| (adjoint.py:98-110)."""
    from paper_1511_03645_b200 import adjoint
    d = FLAG["flag0"]
    p, store = _setup(d)
    for n, t in enumerate(d["interp_t"]):
        w = adjoint.TimeWindow(t, t)   # zero span: exactly the interpolated instant
        _, _, best = adjoint.flag_level([p], t, store, w, np.inf, want_best=True, time_interp=True)
        assert np.array_equal(best[0], d["interp_val"][n])


def test_out_of_range_raises():
    from paper_1511_03645_b200 import adjoint
    from paper_1511_03645_b200.geometry import OutOfRangeError, UniformField
    d = FLAG["flag0"]
    p, store = _setup(d)
    small = [UniformField(values=f.values[:, :10, :], origin=(0.0, 0.0), dx=d["a_dx"], dy=d["a_dy"], time=f.time)
             for f in store.fields]
    st2 = adjoint.AdjointSnapshotStore(times=store.times, fields=small, window=store.window)
    with pytest.raises(OutOfRangeError):
        adjoint.inner_product_field(p, 0.5, st2, st2.window)


def test_empty_window_gives_no_flags():
    """t beyond the last snapshot: query_window_times is empty (adjoint.py:
    192-214) and inner_product_field is zero everywhere (adjoint.py:227-249)."""
    from paper_1511_03645_b200 import adjoint
    d = FLAG["flag0"]
    p, store = _setup(d)
    t = float(d["times"][-1]) + 0.5
    assert adjoint.query_window_times(t, store.window, store) == []
    best = adjoint.inner_product_field(p, t, store, store.window)
    assert not np.any(best)
    ff = adjoint.inner_product_flags(p, t, store, store.window, 0.0)
    assert not ff.flags.any()
    _, counts, _ = adjoint.flag_level([p], t, store, store.window, 0.0)
    assert counts[0] == 0
