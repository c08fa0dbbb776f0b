"""Host-side rectangle-table construction (device.RectTable._split,
device.axis_weight_tables) against straightforward per-rect loops."""
import types

import numpy as np

from paper_1511_03645_b200 import _lib, device


def _loop_split(rects, cap):
    out = []
    for r in rects:
        ni, nj = int(r["ni"]), int(r["nj"])
        if ni * nj <= cap:
            out.append(r.copy())
            continue
        cj = min(nj, cap)
        ci = max(1, cap // cj)
        for a in range(0, ni, ci):
            for b in range(0, nj, cj):
                s = r.copy()
                s["di0"] += a; s["dj0"] += b; s["si0"] += a; s["sj0"] += b
                s["ni"] = min(ci, ni - a); s["nj"] = min(cj, nj - b)
                out.append(s)
    return np.array(out, dtype=_lib.RECT_DTYPE)


def _random_rects(rng, n, kinds=(0, 1, 2)):
    r = np.zeros(n, dtype=_lib.RECT_DTYPE)
    r["kind"] = rng.choice(kinds, n)
    r["dst_patch"] = rng.integers(0, 5, n)
    r["src_patch"] = rng.integers(0, 4, n)
    r["di0"] = rng.integers(0, 8, n)
    r["dj0"] = rng.integers(0, 8, n)
    r["si0"] = rng.integers(0, 8, n)
    r["sj0"] = rng.integers(0, 8, n)
    r["ni"] = rng.integers(1, 70, n)
    r["nj"] = rng.integers(1, 300, n)
    return r


def test_split_matches_loop():
    rng = np.random.default_rng(0)
    for _ in range(20):
        r = _random_rects(rng, 40)
        got = device.RectTable._split(r.copy())
        ref = _loop_split(r, device.RectTable.MAX_CELLS)
        assert got.tobytes() == ref.tobytes()
        assert int((got["ni"] * got["nj"]).max()) <= device.RectTable.MAX_CELLS


def _fake_store(specs, ndim, g):
    pats = [types.SimpleNamespace(spec=types.SimpleNamespace(lo=lo, shape=sh, level=lev)) for lo, sh, lev in specs]
    return types.SimpleNamespace(patches=pats, ndim=ndim, g=g)


def _loop_tables(rects, fs, cs, h):
    level = fs.patches[0].spec.level
    wf, wc, org = h.widths(level), h.widths(level - 1), h.origin
    ws, js, off = [], [], 0
    for r in rects:
        if r["kind"] != _lib.RECT_COARSE:
            continue
        dp = fs.patches[int(r["dst_patch"])].spec
        sp = cs.patches[int(r["src_patch"])].spec
        axes = [(0, int(r["di0"]), int(r["ni"]))] + ([(1, int(r["dj0"]), int(r["nj"]))] if fs.ndim == 2 else [])
        r["pad"] = off
        for ax, d0, n in axes:
            gidx = dp.lo[ax] - fs.g + d0 + np.arange(n)
            coord = org[ax] + (gidx + 0.5) * wf[ax]
            lo_phys = org[ax] + (sp.lo[ax] - cs.g) * wc[ax]
            i0, w = device._axis_weights_np(coord, lo_phys, wc[ax], sp.shape[ax] + 2 * cs.g)
            ws.append(w); js.append(i0.astype(np.int32)); off += n
    return np.concatenate(ws), np.concatenate(js)


def test_axis_weight_tables_match_loop():
    rng = np.random.default_rng(1)
    for ndim in (1, 2):
        widths = {0: (1 / 96, 1 / 80), 1: (1 / 384, 1 / 320)}
        h = types.SimpleNamespace(origin=(-0.25, 0.125), widths=lambda l: widths[l][:ndim])
        fine = [(tuple(rng.integers(0, 300, ndim)), tuple(rng.integers(4, 40, ndim)), 1) for _ in range(5)]
        coarse = [(tuple(rng.integers(0, 70, ndim)), tuple(rng.integers(1, 20, ndim)), 0) for _ in range(4)]
        fs, cs = _fake_store(fine, ndim, 2), _fake_store(coarse, ndim, 2)
        r = _random_rects(rng, 60)
        if ndim == 1:
            r["nj"] = 1
        r1, r2 = r.copy(), r.copy()
        w, i = device.axis_weight_tables(r1, fs, cs, h)
        w0, i0 = _loop_tables(r2, fs, cs, h)
        assert w.tobytes() == w0.tobytes()
        assert np.array_equal(i, i0)
        assert r1.tobytes() == r2.tobytes()


def test_restrict_cells_match_rect_loop():
    """device.restrict_cells flattens restriction rects exactly as k4_restrict
    walks them (amr.py:440-450 order flag from the unsplit overlap box)."""
    rng = np.random.default_rng(2)
    for nd in (1, 2):
        r = 4
        ct = np.zeros(3, dtype=_lib.PATCH_DTYPE)
        ft = np.zeros(4, dtype=_lib.PATCH_DTYPE)
        ct["offset"] = [0, 5000, 9000]
        ct["pitch"] = [12, 20, 8] if nd == 2 else 1
        ft["offset"] = [0, 30000, 70000, 99000]
        ft["pitch"] = [36, 68, 20, 44] if nd == 2 else 1
        cs = types.SimpleNamespace(ndim=nd, g=2, table_np=ct)
        fs = types.SimpleNamespace(ndim=nd, g=2, table_np=ft)
        rects = np.zeros(30, dtype=_lib.RECT_DTYPE)
        rects["dst_patch"] = rng.integers(0, 3, 30)
        rects["src_patch"] = rng.integers(0, 4, 30)
        rects["di0"] = rng.integers(0, 5, 30)
        rects["si0"] = rng.integers(0, 5, 30)
        rects["ni"] = rng.integers(1, 9, 30)
        if nd == 2:
            rects["dj0"] = rng.integers(0, 5, 30)
            rects["sj0"] = rng.integers(0, 5, 30)
            rects["nj"] = rng.choice([1, 2, 7], 30)
        else:
            rects["nj"] = 1
        d, s, m = device.restrict_cells(cs, fs, rects, r)
        want = []
        for R in rects:
            cp, fp = ct[R["dst_patch"]], ft[R["src_patch"]]
            gy = 2 if nd == 2 else 0
            for a in range(R["ni"]):
                for b in range(R["nj"]):
                    cd = cp["offset"] + (2 + R["di0"] + a) * cp["pitch"] + gy + R["dj0"] + b
                    fsrc = fp["offset"] + (2 + R["si0"] + a * r) * fp["pitch"] + gy + R["sj0"] + b * (r if nd == 2 else 1)
                    want.append((cd, fsrc, int(nd == 2 and R["nj"] == 1) | (int(fp["pitch"]) << 1)))
        assert [tuple(map(int, x)) for x in zip(d, s, m)] == want
