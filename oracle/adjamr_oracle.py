"""CPU ORACLE -- test infrastructure only, never the product path.

A numpy restatement of the reference algorithm on the hot path (the
reference is the pure-Python package `adjamr`, /root/reference/pkg/src/
adjamr/*.py; every function below cites the file:line it restates).  It
works on plain arrays in the device layout of include/adjamr_b200.h:

    q    (m, NX, NY)   ghost-inclusive state, y contiguous (1D: (m, NX))
    aux  (naux, NX, NY) material planes: acoustics {c, z, rho, bulk},
                        shallow water {c, depth}

Each operation is evaluated in the reference's order (no fused multiply-add
exists in numpy), so the oracle is bitwise identical to the reference; the
tests pin that against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  Importable only from tests/, bench.py's
cpu_baseline / --impl reference legs and __graft_entry__.smoke().

Exceptions (parity unpinned by the reference): the "periodic" side of
fill_physical is an extension for BASELINE C3 (the reference has wall and
outflow only) and inner_product_interp restates the north_star's
time-interpolated window from adjoint.py:98-110 + 227-249.
"""
from __future__ import annotations

import numpy as np

AC1D, AC2D, SWE2D = "acoustics-1d", "acoustics-2d", "swe-linear-2d"


# ---------------------------------------------------------------------------
# limiter (solver.py:65-77)

def phi(limiter: str, theta):
    if limiter == "none":
        return np.ones_like(theta)
    if limiter == "minmod":
        return np.maximum(0.0, np.minimum(1.0, theta))
    if limiter == "MC":
        return np.maximum(0.0, np.minimum(np.minimum((1.0 + theta) / 2.0, 2.0), 2.0 * theta))
    if limiter == "superbee":
        return np.maximum(0.0, np.maximum(np.minimum(1.0, 2.0 * theta), np.minimum(2.0, theta)))
    raise ValueError(limiter)


def _seqsum(terms):
    """Left-to-right sum, the order numpy uses for a short outer-axis reduction."""
    acc = terms[0]
    for t in terms[1:]:
        acc = acc + t
    return acc


# ---------------------------------------------------------------------------
# interface solves: equations.py:104-349, TimeReversed equations.py:517-531

class Faces:
    """Waves (nw, m, ...), speeds (nw, ...), fluctuations (m, ...) of a batch of faces."""

    def __init__(self, W, s, am, ap, fwave):
        self.W, self.s, self.am, self.ap, self.fwave = W, s, am, ap, fwave


def _fluct(W, s, fwave):
    # _fluctuations / _fwave_fluctuations, equations.py:104-118
    if fwave:
        wn = np.where(s < 0, 1.0, np.where(s == 0, 0.5, 0.0))
        wp = 1.0 - wn
    else:
        wn = np.minimum(s, 0.0)
        wp = np.maximum(s, 0.0)
    am = _seqsum([wn[k][None] * W[k] for k in range(W.shape[0])])
    ap = _seqsum([wp[k][None] * W[k] for k in range(W.shape[0])])
    return am, ap


def _assemble(shape_like, m, comps_per_wave):
    """Stack waves given as {family: {component: array}} (missing = zeros)."""
    nw = len(comps_per_wave)
    W = np.zeros((nw, m, *shape_like.shape))
    for k, comps in enumerate(comps_per_wave):
        for c, v in comps.items():
            W[k, c] = v
    return W


def normal_solve(system, fwave, rev, axis, ql, qr, ml, mr, g=0.0):
    """One batch of interface solves; ml/mr are per-side material planes."""
    mu, mv = 1 + axis, 2 - axis
    m = ql.shape[0]
    if not fwave:
        dq = qr - ql
        if system == AC1D:        # acoustics_rp_1d, equations.py:125-140
            zl, zr = ml[1], mr[1]
            a1 = (-dq[0] + zr * dq[1]) / (zl + zr)
            a2 = (dq[0] + zl * dq[1]) / (zl + zr)
            W = _assemble(a1, m, [{0: -a1 * zl, 1: a1}, {0: a2 * zr, 1: a2}])
            s = np.stack([-ml[0], mr[0]])
        elif system == AC2D:      # acoustics_rp_normal_2d, equations.py:143-169
            zl, zr = ml[1], mr[1]
            a1 = (-dq[0] + zr * dq[mu]) / (zl + zr)
            a2 = (dq[0] + zl * dq[mu]) / (zl + zr)
            W = _assemble(a1, m, [{0: -a1 * zl, mu: a1}, {mv: dq[mv]}, {0: a2 * zr, mu: a2}])
            s = np.stack([-ml[0], np.zeros_like(a1), mr[0]])
        else:                     # swe_linear_rp, equations.py:198-224
            cl, cr = ml[0], mr[0]
            a1 = (cr * dq[0] - dq[mu]) / (cl + cr)
            a2 = (cl * dq[0] + dq[mu]) / (cl + cr)
            W = _assemble(a1, m, [{0: a1, mu: -a1 * cl}, {mv: dq[mv]}, {0: a2, mu: a2 * cr}])
            s = np.stack([-cl, np.zeros_like(a1), cr])
    else:
        # adjoint_flux + adjoint_fwave_rp, equations.py:249-320
        fl = np.zeros_like(ql)
        fr = np.zeros_like(qr)
        if system == AC1D:
            fl[0], fl[1] = ql[1] / ml[2], ml[3] * ql[0]
            fr[0], fr[1] = qr[1] / mr[2], mr[3] * qr[0]
        elif system == AC2D:
            fl[0], fl[mu] = ql[mu] / ml[2], ml[3] * ql[0]
            fr[0], fr[mu] = qr[mu] / mr[2], mr[3] * qr[0]
        else:
            fl[0], fl[mu] = g * ml[1] * ql[mu], ql[0]
            fr[0], fr[mu] = g * mr[1] * qr[mu], qr[0]
        df = fr - fl
        if system == AC1D:
            zl, zr = ml[1], mr[1]
            b1 = (zr * df[0] - df[1]) / (zl + zr)
            b2 = (zl * df[0] + df[1]) / (zl + zr)
            W = _assemble(b1, m, [{0: b1, 1: -b1 * zl}, {0: b2, 1: b2 * zr}])
            s = np.stack([-ml[0], mr[0]])
        elif system == AC2D:
            zl, zr = ml[1], mr[1]
            b1 = (zr * df[0] - df[mu]) / (zl + zr)
            b2 = (zl * df[0] + df[mu]) / (zl + zr)
            W = _assemble(b1, m, [{0: b1, mu: -b1 * zl}, {}, {0: b2, mu: b2 * zr}])
            s = np.stack([-ml[0], np.zeros_like(b1), mr[0]])
        else:
            cl, cr = ml[0], mr[0]
            b1 = (cr * df[mu] - df[0]) / (cl + cr)
            b2 = (cl * df[mu] + df[0]) / (cl + cr)
            W = _assemble(b1, m, [{0: -b1 * cl, mu: b1}, {}, {0: b2 * cr, mu: b2}])
            s = np.stack([-cl, np.zeros_like(b1), cr])
    am, ap = _fluct(W, s, fwave)
    if rev:
        W = -W[::-1] if fwave else W[::-1]
        s = -s[::-1]
        am, ap = -ap, -am
    return Faces(W, s, am, ap, fwave)


def transverse(system, fwave, rev, axis, f, mb, ma, g=0.0):
    """Transverse split (equations.py:172-191, 227-242, 323-349; reversed 529-531).
    mb/ma: planes of the cells below/above; SWE uses the dry-clamped c."""
    mv = 2 - axis
    bm = np.zeros_like(f)
    bp = np.zeros_like(f)
    if system == SWE2D:
        cb = np.sqrt(g * np.where(mb[1] > 0.0, mb[1], 1.0))   # solver.py:383-387
        ca = np.sqrt(g * np.where(ma[1] > 0.0, ma[1], 1.0))
        den = cb + ca
        if not fwave:
            bd = (ca * f[0] - f[mv]) / den
            bu = (cb * f[0] + f[mv]) / den
            bm[0], bm[mv] = -cb * bd, -cb * (-bd * cb)
            bp[0], bp[mv] = ca * bu, ca * (bu * ca)
        else:
            bd = (ca * f[mv] - f[0]) / den
            bu = (cb * f[mv] + f[0]) / den
            bm[0], bm[mv] = -cb * (-bd * cb), -cb * bd
            bp[0], bp[mv] = ca * (bu * ca), ca * bu
    else:
        cb, zb, ca, za = mb[0], mb[1], ma[0], ma[1]
        if not fwave:
            bd = (-f[0] + za * f[mv]) / (zb + za)
            bu = (f[0] + zb * f[mv]) / (zb + za)
            bm[0], bm[mv] = -cb * (-bd * zb), -cb * bd
            bp[0], bp[mv] = ca * (bu * za), ca * bu
        else:
            bd = (za * f[0] - f[mv]) / (zb + za)
            bu = (zb * f[0] + f[mv]) / (zb + za)
            bm[0], bm[mv] = -cb * bd, -cb * (-bd * zb)
            bp[0], bp[mv] = ca * bu, ca * (bu * za)
    if rev:
        return -bp, -bm
    return bm, bp


# ---------------------------------------------------------------------------
# patch step (solver.py:317-512)

def _axis_solve(system, fwave, rev, axis, q, aux, g):
    """_solve_axis (solver.py:390-412) incl. SWE effective states (357-380)."""
    left = [slice(None)] * (q.ndim - 1)
    right = [slice(None)] * (q.ndim - 1)
    left[axis] = slice(None, -1)
    right[axis] = slice(1, None)
    ql, qr = q[(slice(None), *left)], q[(slice(None), *right)]
    ml, mr = aux[(slice(None), *left)], aux[(slice(None), *right)]
    if system != SWE2D:
        return normal_solve(system, fwave, rev, axis, ql, qr, ml, mr, g), None
    mu = 1 + axis
    wl, wr = ml[1] > 0.0, mr[1] > 0.0
    both_wet, both_dry = wl & wr, ~wl & ~wr
    mirror_r = qr.copy()
    mirror_r[mu] *= -1.0
    mirror_l = ql.copy()
    mirror_l[mu] *= -1.0
    qle = np.where(wl, ql, mirror_r)
    qre = np.where(wr, qr, mirror_l)
    dl = np.where(both_dry, 1.0, np.where(wl, ml[1], mr[1]))
    dr = np.where(both_dry, 1.0, np.where(wr, mr[1], ml[1]))
    mle = np.stack([np.sqrt(g * dl), dl])
    mre = np.stack([np.sqrt(g * dr), dr])
    res = normal_solve(system, fwave, rev, axis, qle, qre, mle, mre, g)
    res.W[:, :, both_dry] = 0.0
    res.s[:, both_dry] = 0.0
    res.am[:, both_dry] = 0.0
    res.ap[:, both_dry] = 0.0
    return res, both_wet


def _limited(res: Faces, limiter, axis):
    """_limited_waves (solver.py:317-337): neighbours along the face axis,
    zero beyond the first/last face."""
    W = res.W
    if limiter == "none":
        return W
    ax = 2 + axis
    n = W.shape[ax]
    def shifted(delta):
        out = np.zeros_like(W)
        dst = [slice(None)] * W.ndim
        src = [slice(None)] * W.ndim
        if delta > 0:    # value of face i-1 at position i
            dst[ax], src[ax] = slice(1, n), slice(0, n - 1)
        else:            # value of face i+1 at position i
            dst[ax], src[ax] = slice(0, n - 1), slice(1, n)
        out[tuple(dst)] = W[tuple(src)]
        return out
    up, dn = shifted(1), shifted(-1)
    m = W.shape[1]
    dots = _seqsum([W[:, c] * W[:, c] for c in range(m)])
    d_up = _seqsum([up[:, c] * W[:, c] for c in range(m)])
    d_dn = _seqsum([dn[:, c] * W[:, c] for c in range(m)])
    upwind = np.where(res.s > 0, d_up, d_dn)
    with np.errstate(invalid="ignore", divide="ignore"):
        theta = np.where(dots > 0, upwind / np.where(dots > 0, dots, 1.0), 0.0)
    return phi(limiter, theta)[:, None] * W


def _corr(res: Faces, dtd, limiter, axis):
    """_correction_flux (solver.py:340-348)."""
    lw = _limited(res, limiter, axis)
    a = np.abs(res.s)
    coef = (0.5 * np.sign(res.s)) * (1.0 - dtd * a) if res.fwave else (0.5 * a) * (1.0 - dtd * a)
    return _seqsum([coef[k][None] * lw[k] for k in range(lw.shape[0])])


def step_1d(q, aux, dt, dx, system=AC1D, fwave=False, rev=False, limiter="MC", ghost=2):
    """step_patch_1d (solver.py:415-439); returns (new q, cfl)."""
    q = np.array(q, dtype=float, copy=True)
    g = ghost
    dtdx = dt / dx
    n = q.shape[1]
    res, _ = _axis_solve(system, fwave, rev, 0, q, aux, 0.0)
    cfl = float(np.max(np.abs(res.s[:, g - 1:n - g])) * dtdx) if n > 2 * g else 0.0
    dq = np.zeros_like(q)
    dq[:, 1:] -= dtdx * res.ap
    dq[:, :-1] -= dtdx * res.am
    F = _corr(res, dtdx, limiter, 0)
    dq[:, 1:-1] -= dtdx * (F[:, 1:] - F[:, :-1])
    q[:, g:-g] += dq[:, g:-g]
    return q, cfl


def step_2d(q, aux, dt, dx, dy, system, fwave=False, rev=False, limiter="MC", gravity=0.0, ghost=2):
    """step_patch_2d (solver.py:442-512); returns (new q, cfl)."""
    q = np.array(q, dtype=float, copy=True)
    g = ghost
    dtdx, dtdy = dt / dx, dt / dy
    NX, NY = q.shape[1], q.shape[2]
    swe = system == SWE2D
    rx, wwx = _axis_solve(system, fwave, rev, 0, q, aux, gravity)
    ry, wwy = _axis_solve(system, fwave, rev, 1, q, aux, gravity)
    cfl = max(float(np.max(np.abs(rx.s[:, g - 1:NX - g, g:NY - g]), initial=0.0)) * dtdx,
              float(np.max(np.abs(ry.s[:, g:NX - g, g - 1:NY - g]), initial=0.0)) * dtdy)
    dq = np.zeros_like(q)
    dq[:, 1:, :] -= dtdx * rx.ap
    dq[:, :-1, :] -= dtdx * rx.am
    dq[:, :, 1:] -= dtdy * ry.ap
    dq[:, :, :-1] -= dtdy * ry.am
    F = _corr(rx, dtdx, limiter, 0)
    G = _corr(ry, dtdy, limiter, 1)
    # transverse terms, solver.py:475-496, in the reference's order
    hx = 0.5 * dtdx
    bm, bp = transverse(system, fwave, rev, 0, rx.am[:, :, 1:-1], aux[:, :-1, :-2], aux[:, :-1, 2:], gravity)
    G[:, :-1, 0:NY - 2] -= hx * bm
    G[:, :-1, 1:NY - 1] -= hx * bp
    bm, bp = transverse(system, fwave, rev, 0, rx.ap[:, :, 1:-1], aux[:, 1:, :-2], aux[:, 1:, 2:], gravity)
    G[:, 1:, 0:NY - 2] -= hx * bm
    G[:, 1:, 1:NY - 1] -= hx * bp
    hy = 0.5 * dtdy
    bm, bp = transverse(system, fwave, rev, 1, ry.am[:, 1:-1, :], aux[:, :-2, :-1], aux[:, 2:, :-1], gravity)
    F[:, 0:NX - 2, :-1] -= hy * bm
    F[:, 1:NX - 1, :-1] -= hy * bp
    bm, bp = transverse(system, fwave, rev, 1, ry.ap[:, 1:-1, :], aux[:, :-2, 1:], aux[:, 2:, 1:], gravity)
    F[:, 0:NX - 2, 1:] -= hy * bm
    F[:, 1:NX - 1, 1:] -= hy * bp
    if swe:
        F[:, ~wwx] = 0.0
        G[:, ~wwy] = 0.0
    dq[:, 1:-1, :] -= dtdx * (F[:, 1:, :] - F[:, :-1, :])
    dq[:, :, 1:-1] -= dtdy * (G[:, :, 1:] - G[:, :, :-1])
    if swe:
        dq *= aux[1] > 0.0
    q[:, g:-g, g:-g] += dq[:, g:-g, g:-g]
    return q, cfl


# ---------------------------------------------------------------------------
# ghost fill (solver.py:84-146, 227-286; geometry.py:248-260, 302-327)

def fill_physical(q, ghost, edges, bc, normal_comp):
    """edges/bc: dict side -> bool / 'wall'|'outflow'; sides xlo,xhi,ylo,yhi.
    Slab order x-low, x-high, y-low, y-high (solver.py:136-146)."""
    q = np.array(q, dtype=float, copy=True)
    g = ghost
    for axis, (lo, hi) in enumerate((("xlo", "xhi"), ("ylo", "yhi"))[: q.ndim - 1]):
        ax = 1 + axis
        n = q.shape[ax]
        for side, high in ((lo, False), (hi, True)):
            if not edges.get(side, False):
                continue
            if bc[side] == "periodic":   # extension (no reference counterpart): wrap to the opposite interior
                src_idx = np.arange(g, 2 * g) if high else np.arange(n - 2 * g, n - g)
            else:
                src_idx = (np.arange(n - g - 1, n - 2 * g - 1, -1) if high else np.arange(2 * g - 1, g - 1, -1)) \
                    if bc[side] == "wall" else np.full(g, n - g - 1 if high else g)
            dst_idx = np.arange(n - g, n) if high else np.arange(0, g)
            vals = np.take(q, src_idx, axis=ax)
            if bc[side] == "wall":
                vals[normal_comp[axis]] *= -1.0
            sl = [slice(None)] * q.ndim
            sl[ax] = dst_idx
            q[tuple(sl)] = vals
    return q


def axis_weights(coord, origin, width, n):
    """_axis_weights (geometry.py:248-260)."""
    s = (np.asarray(coord, dtype=float) - origin) / width - 0.5
    i0 = np.floor(s).astype(int)
    w = s - i0
    w = np.where(i0 < 0, 0.0, np.where(i0 > n - 2, 1.0, w))
    i0 = np.clip(i0, 0, max(n - 2, 0))
    if n == 1:
        w = np.zeros_like(w)
    return i0, w


def bilinear(v, i0, j0, wx, wy):
    """interpolate_uniform / interpolate_patch arithmetic (geometry.py:287-290, 324-327)."""
    nx, ny = v.shape[1], v.shape[2]
    i1 = np.minimum(i0 + 1, nx - 1)
    j1 = np.minimum(j0 + 1, ny - 1)
    return (v[:, i0, j0] * (1 - wx) * (1 - wy) + v[:, i1, j0] * wx * (1 - wy)
            + v[:, i0, j1] * (1 - wx) * wy + v[:, i1, j1] * wx * wy)


def linear(v, i0, wx):
    n = v.shape[1]
    return v[:, i0] * (1 - wx) + v[:, np.minimum(i0 + 1, n - 1)] * wx


def coarse_interp(cstate_old, cstate_new, clo, cghost, cdx, origin, fine_idx, fdx, w_time, mode):
    """space_time_interp + interpolate_patch (solver.py:266-286, geometry.py:302-327)
    at fine global cell indices fine_idx (tuple of int arrays).
    mode 0: old only, 1: blend, 2: new only."""
    nd = len(fine_idx)
    pts = [origin[a] + (fine_idx[a] + 0.5) * fdx[a] for a in range(nd)]
    lo_phys = [origin[a] + (clo[a] - cghost) * cdx[a] for a in range(nd)]
    shape = cstate_new.shape[1:]
    iw = [axis_weights(pts[a], lo_phys[a], cdx[a], shape[a]) for a in range(nd)]

    def ev(v):
        return linear(v, *iw[0]) if nd == 1 else bilinear(v, iw[0][0], iw[1][0], iw[0][1], iw[1][1])
    if mode == 0:
        return ev(cstate_old)
    if mode == 2:
        return ev(cstate_new)
    return (1.0 - w_time) * ev(cstate_old) + w_time * ev(cstate_new)


def time_mode(t, t0, t1, has_old):
    """Scheduling rules of space_time_interp (solver.py:269-286): (mode, w) or raise."""
    t_cur = t1
    eps = 1e-9 * max(abs(t_cur), 1.0)
    if not has_old:
        if abs(t - t_cur) > eps:
            raise RuntimeError("scheduling")
        return 2, 1.0
    if not t0 - eps <= t <= t1 + eps:
        raise RuntimeError("scheduling")
    if t1 == t0:
        return 0, 0.0
    w = float(np.clip((t - t0) / (t1 - t0), 0.0, 1.0))
    if w == 0.0:
        return 0, 0.0
    return 1, w


# ---------------------------------------------------------------------------
# restriction (amr.py:399-450)

def restrict_block(fine_block, ratio, ndim, wet_f=None, wet_c=None, coarse_cur=None):
    """Mean of r (x r) children; fine_block (m, nx*r[, ny*r]) interior data.
    SWE: wet-weighted mean written only where wet_c and any wet child."""
    m = fine_block.shape[0]
    if ndim == 1:
        blocks = fine_block.reshape(m, -1, ratio)
        if wet_f is None:
            return blocks.mean(axis=2)
        w = wet_f.reshape(-1, ratio).astype(float)
        ws = w.sum(axis=1)
        avg = (blocks * w).sum(axis=2) / np.where(ws > 0, ws, 1.0)
    else:
        nxc, nyc = fine_block.shape[1] // ratio, fine_block.shape[2] // ratio
        blocks = fine_block.reshape(m, nxc, ratio, nyc, ratio)
        if wet_f is None:
            return blocks.mean(axis=(2, 4))
        w = wet_f.reshape(nxc, ratio, nyc, ratio).astype(float)
        ws = w.sum(axis=(1, 3))
        avg = (blocks * w).sum(axis=(2, 4)) / np.where(ws > 0, ws, 1.0)
    out = np.array(coarse_cur, copy=True)
    take = (ws > 0) & wet_c
    out[:, take] = avg[:, take]
    return out


# ---------------------------------------------------------------------------
# adjoint flagging (adjoint.py:98-110, 192-257; geometry.py:263-290)

def window_indices(t, span, t_final, times):
    """query_window_times (adjoint.py:192-214)."""
    times = np.asarray(times, dtype=float)
    dts = float(times[1] - times[0]) if len(times) > 1 else 0.0
    eps = 1e-9 * max(dts, abs(float(times[-1])), 1.0)
    if t > times[-1] + eps:
        return []
    upper = min(t + span, t_final)
    inside = [int(k) for k in np.nonzero((times >= t - eps) & (times <= upper + eps))[0]]
    out = list(inside)
    if not inside or times[inside[0]] > t + eps:
        below = np.nonzero(times < t - eps)[0]
        if len(below):
            out.insert(0, int(below[-1]))
    if not inside or times[inside[-1]] < upper - eps:
        above = np.nonzero(times > upper + eps)[0]
        if len(above):
            out.append(int(above[0]))
    return out


def uniform_sample(values, origin, dx, dy, x, y=None):
    """interpolate_uniform (geometry.py:263-290) incl. its bounds check."""
    shape = values.shape[1:]
    hi0 = origin[0] + shape[0] * dx
    eps = 1e-12 * max(abs(hi0 - origin[0]), 1.0)
    x = np.asarray(x, dtype=float)
    if np.any(x < origin[0] - eps) or np.any(x > hi0 + eps):
        raise IndexError("interpolation point outside domain in x")
    i0, wx = axis_weights(x, origin[0], dx, shape[0])
    if y is None:
        return linear(values, i0, wx)
    hi1 = origin[1] + shape[1] * dy
    y = np.asarray(y, dtype=float)
    if np.any(y < origin[1] - eps) or np.any(y > hi1 + eps):
        raise IndexError("interpolation point outside domain in y")
    j0, wy = axis_weights(y, origin[1], dy, shape[1])
    return bilinear(values, i0, j0, wx, wy)


def inner_product(q_int, xc, yc, fields, idx, a_origin, a_dx, a_dy, fwd_wet=None, adj_wet=None):
    """inner_product_field (adjoint.py:227-249): windowed max of |qhat . q|.
    q_int (m, nx[, ny]) interior; xc/yc cell-centre grids; fields (N, m, ...)."""
    best = np.zeros(q_int.shape[1:])
    for k in idx:
        qh = uniform_sample(fields[k], a_origin, a_dx, a_dy, xc, yc)
        best = np.maximum(best, np.abs(_seqsum([qh[c] * q_int[c] for c in range(q_int.shape[0])])))
    if fwd_wet is not None:
        best = np.where(fwd_wet, best, 0.0)
    if adj_wet is not None and yc is not None:
        shape = adj_wet.shape
        i = np.clip(((xc - a_origin[0]) / a_dx).astype(int), 0, shape[0] - 1)
        j = np.clip(((yc - a_origin[1]) / a_dy).astype(int), 0, shape[1] - 1)
        best = np.where(~adj_wet[i, j], 0.0, best)
    return best


def inner_product_interp(q_int, xc, yc, fields, times, t_eval, a_origin, a_dx, a_dy):
    """Time-interpolated mode: AdjointSnapshotStore.interpolate_time
    (adjoint.py:98-110) at each t in t_eval, then |qhat . q|, max."""
    times = np.asarray(times, dtype=float)
    eps = 1e-9 * max(abs(times[-1]), 1.0)
    best = np.zeros(q_int.shape[1:])
    for t in t_eval:
        if t <= times[0] + eps:
            vals = fields[0]
        elif t >= times[-1] - eps:
            vals = fields[-1]
        else:
            n = int(np.searchsorted(times, t) - 1)
            w = (t - times[n]) / (times[n + 1] - times[n])
            vals = (1 - w) * fields[n] + w * fields[n + 1]
        qh = uniform_sample(vals, a_origin, a_dx, a_dy, xc, yc)
        best = np.maximum(best, np.abs(_seqsum([qh[c] * q_int[c] for c in range(q_int.shape[0])])))
    return best


# ---------------------------------------------------------------------------
# output path

def interpolate_time(fields, times, t):
    """AdjointSnapshotStore.interpolate_time (adjoint.py:98-110) on arrays."""
    times = np.asarray(times, dtype=float)
    eps = 1e-9 * max(abs(times[-1]), 1.0)
    if t <= times[0] + eps:
        return fields[0]
    if t >= times[-1] - eps:
        return fields[-1]
    n = int(np.searchsorted(times, t) - 1)
    w = (t - times[n]) / (times[n + 1] - times[n])
    return (1 - w) * fields[n] + w * fields[n + 1]


def evaluate_J(levels, ratios, origin, widths, qhat, a_origin, a_dx, a_dy):
    """evaluate_J on a hierarchy (adjoint.py:299-336) with _uncovered_mask
    (adjoint.py:280-296).  levels[l] = list of (lo, interior q (m, nx[, ny]));
    widths[l] = (wx, wy) of level l+1; qhat = the (time-interpolated) adjoint
    field values (m, nxa[, nya])."""
    nd = len(origin)
    total = 0.0
    for li, plist in enumerate(levels):
        wx, wy = widths[li]
        area = wx if nd == 1 else wx * wy
        finer = levels[li + 1] if li + 1 < len(levels) else []
        for lo, q in plist:
            shape = q.shape[1:]
            hi = tuple(l + n - 1 for l, n in zip(lo, shape))
            keep = np.ones(shape, dtype=bool)
            if finer:
                r = ratios[li]
                for flo, fq in finer:
                    fhi = tuple(l + n - 1 for l, n in zip(flo, fq.shape[1:]))
                    clo = tuple(max(flo[a] // r, lo[a]) for a in range(nd))
                    chi = tuple(min(fhi[a] // r, hi[a]) for a in range(nd))
                    if any(a > b for a, b in zip(clo, chi)):
                        continue
                    keep[tuple(slice(a - l, b - l + 1) for a, b, l in zip(clo, chi, lo))] = False
            cs = [origin[a] + (np.arange(lo[a], hi[a] + 1) + 0.5) * (wx, wy)[a] for a in range(nd)]
            if nd == 1:
                qh = uniform_sample(qhat, a_origin, a_dx, a_dy, cs[0])
            else:
                x = np.broadcast_to(cs[0][:, None], shape)
                y = np.broadcast_to(cs[1][None, :], shape)
                qh = uniform_sample(qhat, a_origin, a_dx, a_dy, x, y)
            prod = np.sum(qh * q, axis=0)
            total += float(np.sum(prod[keep]) * area)
    return total


def gauge_value(q_int, lo, origin, widths, point):
    """interpolate_patch(interior_only=True) (geometry.py:302-327) at one point
    of a patch's interior q (m, nx[, ny]) -- what record_gauge stores."""
    nd = len(lo)
    shape = q_int.shape[1:]
    lo_phys = [origin[a] + lo[a] * widths[a] for a in range(nd)]
    i0, wx = axis_weights(np.array([point[0]]), lo_phys[0], widths[0], shape[0])
    if nd == 1:
        return (q_int[:, i0] * (1 - wx) + q_int[:, np.minimum(i0 + 1, shape[0] - 1)] * wx)[:, 0]
    j0, wy = axis_weights(np.array([point[1]]), lo_phys[1], widths[1], shape[1])
    i1 = np.minimum(i0 + 1, shape[0] - 1)
    j1 = np.minimum(j0 + 1, shape[1] - 1)
    return (q_int[:, i0, j0] * (1 - wx) * (1 - wy) + q_int[:, i1, j0] * wx * (1 - wy)
            + q_int[:, i0, j1] * (1 - wx) * wy + q_int[:, i1, j1] * wx * wy)[:, 0]


def finest_patch_at(levels, origin, widths, level_shapes, point):
    """PatchHierarchy.finest_patch_at (geometry.py:197-215): (level index,
    patch index) of the finest patch containing the point, lowest index wins."""
    found = None
    for li, plist in enumerate(levels):
        cell = tuple(int(np.clip(np.floor((point[a] - origin[a]) / widths[li][a]), 0, level_shapes[li][a] - 1))
                     for a in range(len(origin)))
        for k, (lo, q) in enumerate(plist):
            hi = tuple(l + n - 1 for l, n in zip(lo, q.shape[1:]))
            if all(l <= c <= h for l, c, h in zip(lo, cell, hi)):
                found = (li, k)
                break
    return found
