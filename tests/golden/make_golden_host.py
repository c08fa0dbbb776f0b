"""Golden vectors for the host-side AMR bookkeeping (clustering, buffering,
nesting), produced by the REFERENCE (build container only):
    python tests/golden/make_golden_host.py  -> tests/golden/host.npz
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from adjamr import amr as ramr          # noqa: E402
from adjamr import geometry as rgeo     # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def blobs(rng, shape):
    m = np.zeros(shape, bool)
    for _ in range(rng.integers(1, 5)):
        c = [rng.integers(0, s) for s in shape]
        r = [rng.integers(1, max(2, s // 3)) for s in shape]
        sl = tuple(slice(max(0, ci - ri), ci + ri) for ci, ri in zip(c, r))
        m[sl] = True
    m ^= rng.random(shape) < rng.choice([0.0, 0.02, 0.1])
    return m


def main():
    rng = np.random.default_rng(7)
    out = {}
    for k in range(160):
        nd = 1 if k % 5 == 0 else 2
        shape = (int(rng.integers(4, 70)),) if nd == 1 else (int(rng.integers(3, 50)), int(rng.integers(3, 50)))
        mask = blobs(rng, shape)
        eff = float(rng.choice([0.5, 0.7, 0.85, 1.0]))
        max_edge = [None, 4, 8, 16, 30][k % 5]
        boxes = ramr.cluster(mask, eff, max_edge=max_edge)
        buf = int(rng.integers(0, 4))
        ff = ramr.FlagField(flags=mask, lo=(0,) * nd, level=1, strategy_name="x", time=0.0)
        bf = ramr.buffer_flags(ff, buf).flags
        allowed = ~blobs(rng, shape) | (rng.random(shape) < 0.5)
        rects = []
        for b in boxes:
            rects += ramr._allowed_rectangles(b, allowed, mask & allowed)
        out[f"c{k}.mask"] = mask
        out[f"c{k}.eff"] = np.array(eff)
        out[f"c{k}.max_edge"] = np.array(-1 if max_edge is None else max_edge)
        out[f"c{k}.boxes"] = np.array([[*b.lo, *b.hi, b.efficiency] for b in boxes], dtype=float).reshape(-1, 2 * nd + 1)
        out[f"c{k}.buf"] = np.array(buf)
        out[f"c{k}.buffered"] = bf
        out[f"c{k}.allowed"] = allowed
        out[f"c{k}.rects"] = np.array([[*b.lo, *b.hi, b.efficiency] for b in rects], dtype=float).reshape(-1, 2 * nd + 1)
    # nesting masks on random hierarchies
    for k in range(20):
        h = rgeo.PatchHierarchy(xlim=(0, 1), ylim=(0, 1), base_shape=(16, 12), ratios=[2])
        ps = []
        for _ in range(rng.integers(1, 4)):
            lo = (int(rng.integers(0, 12)), int(rng.integers(0, 8)))
            hi = (int(lo[0] + rng.integers(0, 5)), int(lo[1] + rng.integers(0, 5)))
            hi = (min(hi[0], 15), min(hi[1], 11))
            if any(rgeo.patches_overlap(rgeo.PatchSpec(1, lo, hi, 1, 1, (0, 0)), q.spec) for q in ps):
                continue
            ps.append(rgeo.Patch(h.make_spec(1, lo, hi), 3))
        h.levels = [ps]
        out[f"n{k}.boxes"] = np.array([[*p.spec.lo, *p.spec.hi] for p in ps])
        out[f"n{k}.allowed"] = rgeo.allowed_region_mask(h, 1)
    path = os.path.join(OUT, "host.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()
