"""Shared helpers: build product patches/equations from golden fixtures."""
import numpy as np

from paper_1511_03645_b200 import equations as E
from paper_1511_03645_b200.geometry import Patch, PatchHierarchy


def dummy_model(name, gravity=9.81):
    if name.startswith("swe"):
        return E.SweMaterialModel(lambda x, y: np.zeros_like(np.asarray(x, float)) - 1.0, gravity=gravity)
    return E.AcousticsMaterialModel(lambda x, y=None: np.ones_like(np.asarray(x, float)),
                                    lambda x, y=None: np.ones_like(np.asarray(x, float)))


def make_equation(name, gravity=9.81):
    m = dummy_model(name, gravity)
    table = {
        "ac2d": lambda: E.Acoustics2D(m),
        "ac2d_adj_rev": lambda: E.Acoustics2D(m).adjoint().reversed(),
        "ac2d_adj": lambda: E.Acoustics2D(m).adjoint(),
        "ac2d_rev": lambda: E.TimeReversed(E.Acoustics2D(m)),
        "swe_wet": lambda: E.SweLinear2D(m),
        "swe_dry": lambda: E.SweLinear2D(m),
        "swe_adj_rev": lambda: E.SweLinear2D(m).adjoint().reversed(),
        "swe_wet_adj_rev": lambda: E.SweLinear2D(m).adjoint().reversed(),
        "ac1d": lambda: E.Acoustics1D(m),
        "ac1d_adj_rev": lambda: E.Acoustics1D(m).adjoint().reversed(),
    }
    return table[name]()


def material_from_planes(aux, swe, gravity=9.81):
    if swe:
        depth = aux[1]
        return E.SweMaterial(bathymetry=-depth, depth=depth, wet=depth > 0, c=aux[0], gravity=gravity)
    return E.AcousticsMaterial(bulk=aux[3], rho=aux[2], c=aux[0], z=aux[1])


def patch_from_arrays(q, aux, swe, dx, dy, lo=None, gravity=9.81, level=1):
    nd = q.ndim - 1
    shape = tuple(n - 4 for n in q.shape[1:])
    lo = lo if lo is not None else (0,) * nd
    xlim = (0.0, dx * shape[0])
    ylim = None if nd == 1 else (0.0, dy * shape[1])
    h = PatchHierarchy(xlim=xlim, ylim=ylim, base_shape=shape, ratios=[])
    spec = h.make_spec(level, lo, tuple(l + n - 1 for l, n in zip(lo, shape)))
    p = Patch(spec, q.shape[0])
    p.aux = material_from_planes(aux, swe, gravity)
    p.state = np.array(q, copy=True)
    return h, p


def norm_rel(a, b):
    """max|a-b| / max|b| per component, maximum over components."""
    out = 0.0
    for c in range(b.shape[0]):
        den = np.max(np.abs(b[c]))
        num = np.max(np.abs(a[c] - b[c]))
        out = max(out, num / den if den > 0 else num)
    return out
