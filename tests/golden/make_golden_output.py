"""Golden values for the output path by running the REFERENCE:
evaluate_J (adjoint.py:299-336) in its store and phi forms and record_gauge
(runio.py:217-226), on the reference's own AMR hierarchies after the first
coarse step of the golden AMR runs (tests/golden/amr.npz).

Run in the build container (needs /root/reference):
    python tests/golden/make_golden_output.py   -> tests/golden/output.npz
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from adjamr import adjoint as radj   # noqa: E402
from adjamr import geometry as rgeo  # noqa: E402
from adjamr import runio as rio      # noqa: E402

from tests.amr_cases import CASES    # noqa: E402
from tests.golden_io import load     # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
NAMES = ("ac2d_adjoint", "ac2d_hetero", "ac1d_adjoint")


def hierarchy(name, g):
    """The reference hierarchy after coarse step 0 (all levels at t = dt)."""
    case = CASES[name]
    h = rgeo.PatchHierarchy(xlim=case["xlim"], ylim=case.get("ylim"), base_shape=case["base"],
                            ratios=list(case["ratios"]))
    t = float(g["dt"])
    h.levels = []
    for lev in range(1, int(g["s0_nlev"]) + 1):
        boxes, q = g[f"s0_L{lev}_boxes"], g[f"s0_L{lev}_q"]
        nd = boxes.shape[1] // 2
        ps, off = [], 0
        for b in boxes:
            lo, hi = tuple(int(v) for v in b[:nd]), tuple(int(v) for v in b[nd:])
            shape = tuple(hh - ll + 1 for ll, hh in zip(lo, hi))
            p = rgeo.Patch(h.make_spec(lev, lo, hi), q.shape[0], time=t)
            n = int(np.prod(shape))
            p.interior()[...] = q[:, off:off + n].reshape(q.shape[0], *shape)
            off += n
            ps.append(p)
        h.levels.append(ps)
    return h, t


def store_of(name, g):
    case = CASES[name]
    nd = case["ndim"]
    origin = (case["xlim"][0],) if nd == 1 else (case["xlim"][0], case["ylim"][0])
    shp = case["adjoint_shape"]
    dx = (case["xlim"][1] - case["xlim"][0]) / shp[0]
    dy = 0.0 if nd == 1 else (case["ylim"][1] - case["ylim"][0]) / shp[1]
    fields = [rgeo.UniformField(values=v, origin=origin, dx=dx, dy=dy, time=t)
              for v, t in zip(g["store_fields"], g["store_times"])]
    return radj.AdjointSnapshotStore(times=g["store_times"], fields=fields,
                                     window=radj.TimeWindow(*case["window"]))


def main():
    amr = load("amr.npz")
    rng = np.random.default_rng(11)
    out = {}
    for name in NAMES:
        g = amr[name]
        case = CASES[name]
        h, t = hierarchy(name, g)
        st = store_of(name, g)
        times = np.asarray(st.times)
        tl = [float(times[0]), t, 0.5 * (times[1] + times[2]), float(times[-1]) - 0.3 * (times[-1] - times[-2]),
              float(times[-1]) + 1.0]
        out[f"{name}.J_times"] = np.array(tl)
        out[f"{name}.J_store"] = np.array([radj.evaluate_J(h, st, tt) for tt in tl])
        out[f"{name}.J_phi"] = np.array([radj.evaluate_J(h, st.fields[-1], tt) for tt in tl[:1]])
        # gauges anywhere in the domain (the finest cover holds them)
        nd = case["ndim"]
        xs = rng.uniform(*case["xlim"], size=12)
        locs = xs[:, None] if nd == 1 else np.stack([xs, rng.uniform(*case["ylim"], size=12)], axis=1)
        vals, found = [], []
        for k, loc in enumerate(locs):
            s = rio.GaugeSeries(gauge_id=k, location=tuple(float(v) for v in loc))
            rio.record_gauge(h, s, t)
            found.append(bool(s.values))
            vals.append(s.values[0] if s.values else np.full(2 if nd == 1 else 3, np.nan))
        out[f"{name}.gauge_locs"] = locs
        out[f"{name}.gauge_vals"] = np.array(vals)
        out[f"{name}.gauge_found"] = np.array(found)
        out[f"{name}.t"] = np.array(t)
        print(name, out[f"{name}.J_store"], out[f"{name}.J_phi"], int(np.sum(found)))
    np.savez(os.path.join(OUT, "output.npz"), **out)


if __name__ == "__main__":
    main()
