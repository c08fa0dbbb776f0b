"""Pin the CPU oracle against the reference's own outputs (bitwise)."""
import numpy as np
import pytest

from oracle import adjamr_oracle as O
from tests.golden_io import SYSTEMS, load

STEP = load("step.npz")
GHOST = load("ghost.npz")
RESTRICT = load("restrict.npz")
FLAG = load("flag.npz")
INTEG = load("integrate.npz")


@pytest.mark.parametrize("case", sorted(STEP))
def test_step_bitwise(case):
    d = STEP[case]
    system, fw, rev = SYSTEMS[d["name"]]
    if system == O.AC1D:
        q, cfl = O.step_1d(d["q_in"], d["aux"], d["dt"], d["dx"], system, fw, rev, d["limiter"])
    else:
        q, cfl = O.step_2d(d["q_in"], d["aux"], d["dt"], d["dx"], d["dy"], system, fw, rev, d["limiter"], d["gravity"])
    assert np.array_equal(q, d["q_out"]), np.max(np.abs(q - d["q_out"]))
    assert cfl == d["cfl"]


def _edges(lo, shape, level_shape):
    e = {"xlo": lo[0] == 0, "xhi": lo[0] + shape[0] == level_shape[0]}
    if len(lo) == 2:
        e.update(ylo=lo[1] == 0, yhi=lo[1] + shape[1] == level_shape[1])
    return e


def _bc(arr):
    return dict(zip(("xlo", "xhi", "ylo", "yhi"), [str(s) for s in arr]))


@pytest.mark.parametrize("case", [c for c in sorted(GHOST) if c.startswith("phys")])
def test_physical_fill_bitwise(case):
    d = GHOST[case]
    q = O.fill_physical(d["q_in"], 2, _edges(d["lo"], d["shape"], d["level_shape"]), _bc(d["bc"]), (1, 2))
    assert np.array_equal(q, d["q_out"])


def test_integrate_sequence_bitwise():
    for case, d in INTEG.items():
        system, fw, rev = SYSTEMS[d["name"]]
        q = d["q0"].copy()
        nd = q.ndim - 1
        shape = tuple(n - 4 for n in q.shape[1:])
        edges = _edges((0,) * nd, shape, shape)
        c = d["aux"][0]
        g = 2
        inner = c[g:-g, g:-g] if nd == 2 else c[g:-g]
        dx, dy = d["dx"], d["dy"]
        base = 0.9 * dx / float(np.max(inner))
        if nd == 2:
            base = min(base, 0.9 * dy / float(np.max(inner)))
        t, n = 0.0, 0
        eps = 1e-9 * max(abs(d["t_end"]), 1.0)
        while t < d["t_end"] - eps:
            dt = min(base, d["t_end"] - t)
            q = O.fill_physical(q, 2, edges, _bc(d["bc"]), (1, 2) if nd == 2 else (1,))
            if nd == 1:
                q, _ = O.step_1d(q, d["aux"], dt, dx, system, fw, rev, "MC")
            else:
                q, _ = O.step_2d(q, d["aux"], dt, dx, dy, system, fw, rev, "MC", d["gravity"])
            t += dt
            n += 1
        assert n == d["nsteps"]
        g2 = (slice(None),) + (slice(2, -2),) * nd
        assert np.array_equal(q[g2], d["q_out"][g2]), case


def test_coarse_interp_bitwise():
    d = GHOST["coarse0"]
    origin = (0.0, 0.0)
    cdx = (2.0 / 16, 1.5 / 12)
    fdx = (cdx[0] / 2, cdx[1] / 2)
    flo, fhi = (10, 6), (21, 17)
    g = 2
    ii, jj = np.meshgrid(np.arange(flo[0] - g, fhi[0] + g + 1), np.arange(flo[1] - g, fhi[1] + g + 1), indexing="ij")
    ghost = ~((ii >= flo[0]) & (ii <= fhi[0]) & (jj >= flo[1]) & (jj <= fhi[1]))
    indom = ghost & (ii >= 0) & (ii < 32) & (jj >= 0) & (jj < 24)
    for n, t in enumerate(d["t_list"]):
        want = d[f"f_t{n}"]
        got = np.zeros_like(want)
        mode, w = O.time_mode(t, 0.0, 0.4, True)
        for clo, old, new in (((0, 0), d["c0_old"], d["c0_new"]), ((8, 0), d["c1_old"], d["c1_new"])):
            chi = (clo[0] + 7, 11)
            sel = indom & (ii // 2 >= clo[0]) & (ii // 2 <= chi[0]) & (jj // 2 >= clo[1]) & (jj // 2 <= chi[1])
            vals = O.coarse_interp(old, new, clo, g, cdx, origin, (ii[sel], jj[sel]), fdx, w, mode)
            got[:, sel] = vals
        assert np.array_equal(got[:, indom], want[:, indom])


@pytest.mark.parametrize("case", sorted(RESTRICT))
def test_restrict_bitwise(case):
    d = RESTRICT[case]
    r = int(d["ratio"])
    swe = str(d["name"]).startswith("swe")
    c = d["c_in"].copy()
    g = 2
    for k in (0, 1):
        f = d[f"f{k}"]
        lo = d["f_lohi"][k][:2]
        hi = d["f_lohi"][k][2:]
        clo, chi = lo // r, hi // r
        fint = f[:, g:-g, g:-g]
        csl = (slice(None), slice(g + clo[0], g + chi[0] + 1), slice(g + clo[1], g + chi[1] + 1))
        if swe:
            wet_f = d[f"f{k}_aux"][1][g:-g, g:-g] > 0
            wet_c = d["c_aux"][1][csl[1:]] > 0
            c[csl] = O.restrict_block(fint, r, 2, wet_f, wet_c, c[csl])
        else:
            c[csl] = O.restrict_block(fint, r, 2)
    assert np.array_equal(c, d["c_out"])


def _centers(lo, shape, dx, dy):
    x = (np.arange(lo[0], lo[0] + shape[0]) + 0.5) * dx
    y = (np.arange(lo[1], lo[1] + shape[1]) + 0.5) * dy
    return np.broadcast_to(x[:, None], tuple(shape)), np.broadcast_to(y[None, :], tuple(shape))


@pytest.mark.parametrize("case", ["flag0", "flag1", "flag2"])
def test_flag_bitwise(case):
    d = FLAG[case]
    lo, shape = d["lo"], d["shape"]
    xc, yc = _centers(lo, shape, d["dx"], d["dy"])
    qi = d["q"][:, 2:-2, 2:-2]
    swe = str(d["name"]).startswith("swe")
    fwd_wet = d["aux"][1][2:-2, 2:-2] > 0 if swe else None
    adj_wet = d["adj_wet"] if d["adj_wet"].size else None
    for n, t in enumerate(d["t_list"]):
        idx = O.window_indices(t, 1.0, 2.0, d["times"])
        assert idx == list(d[f"idx{n}"])
        best = O.inner_product(qi, xc, yc, d["fields"], idx, (0.0, 0.0), d["a_dx"], d["a_dy"], fwd_wet, adj_wet)
        assert np.array_equal(best, d[f"best{n}"])
        assert np.array_equal(best > d["tol"], d[f"flags{n}"])
    vals = O.inner_product_interp(qi, xc, yc, d["fields"], d["times"], [0.37], (0.0, 0.0), d["a_dx"], d["a_dy"])
    assert np.array_equal(vals, d["interp_val"][0])


def test_flag_1d_bitwise():
    d = FLAG["flag1d"]
    x = (np.arange(10, 60) + 0.5) * d["dx"]
    best = O.inner_product(d["q"][:, 2:-2], x, None, d["fields"], list(d["idx"]), (0.0,), d["a_dx"], 0.0)
    assert np.array_equal(best, d["best"])


def test_window_queries():
    d = FLAG["window"]
    for k in range(len(d["t"])):
        n = d["ntimes"][k]
        got = O.window_indices(d["t"][k], d["tf"][k] - d["ts"][k], d["tf"][k], d["times"][k][:n])
        want = [int(v) for v in d["idx"][k] if v >= 0]
        assert got == want
        if got:   # the windows are always a contiguous index range
            assert got == list(range(got[0], got[-1] + 1))
