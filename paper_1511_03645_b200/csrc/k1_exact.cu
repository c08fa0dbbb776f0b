// K1, EXACT variant: one thread per interior cell, every face quantity
// recomputed in the reference's expression order.  This translation unit is
// compiled with -fmad=false so no multiply-add is contracted, making the
// result bitwise identical to the numpy reference (IEEE binary64, correctly
// rounded +,-,*,/,sqrt).  It is the parity anchor for the FAST variant.
//
// Reference (paths under /root/reference/pkg/src/adjamr/):
//   step_patch_1d / step_patch_2d   solver.py:415-512
//   _solve_axis / SWE wet-dry       solver.py:351-412
//   _limited_waves / _correction_flux / limiter_phi  solver.py:65-77, 317-348
//   Riemann + transverse solvers    equations.py:104-349
//   TimeReversed                    equations.py:496-534
#include "adj_common.cuh"

// inlining of the per-face helpers: out of line they pass their arrays
// through local memory (760-830 B of stack per thread); inlined: 202
// registers, no stack, C4 19.5 -> 6.7 ms per step (bitwise unchanged)
#ifndef K1X_INLINE_FACE
#define K1X_INLINE_FACE 1
#endif
#ifndef K1X_INLINE_TIL
#define K1X_INLINE_TIL 1
#endif
#if K1X_INLINE_FACE
#define K1X_FACE_INL __forceinline__
#else
#define K1X_FACE_INL __noinline__
#endif
#if K1X_INLINE_TIL
#define K1X_TIL_INL __forceinline__
#else
#define K1X_TIL_INL __noinline__
#endif

namespace adj {
namespace exact {

struct Rp {
    double w[3][3];  // [family][component]
    double s[3];
    double am[3];
    double ap[3];
};

template <int SYS, int FORM, bool REV>
struct Step {
    static constexpr int M = (SYS == ADJ_SYS_AC1D) ? 2 : 3;
    static constexpr int NW = (SYS == ADJ_SYS_AC1D) ? 2 : 3;
    static constexpr bool SWE = (SYS == ADJ_SYS_SWE2D);
    static constexpr bool FW = (FORM == ADJ_FORM_FWAVE);

    // _fluctuations / _fwave_fluctuations (equations.py:104-118)
    static ADJ_D void fluct(Rp& r) {
        for (int c = 0; c < M; ++c) {
            double am = 0.0, ap = 0.0;
            for (int k = 0; k < NW; ++k) {
                double wn, wp;
                if (FW) {
                    wn = r.s[k] < 0.0 ? 1.0 : (r.s[k] == 0.0 ? 0.5 : 0.0);
                    wp = 1.0 - wn;
                } else {
                    wn = fmin(r.s[k], 0.0);
                    wp = fmax(r.s[k], 0.0);
                }
                if (k == 0) { am = wn * r.w[k][c]; ap = wp * r.w[k][c]; }
                else { am = am + wn * r.w[k][c]; ap = ap + wp * r.w[k][c]; }
            }
            r.am[c] = am;
            r.ap[c] = ap;
        }
    }

    // Normal solve from (effective) states; materials per side.
    //   acoustics: m0=c, m1=z, m2=rho, m3=bulk ; swe: m0=c, m1=depth
    static ADJ_D void normal(int axis, const double* ql, const double* qr,
                             const double* ml, const double* mr, double g, Rp& r) {
        const int mu = 1 + axis, mv = 2 - axis;
        for (int k = 0; k < 3; ++k) { r.s[k] = 0.0; for (int c = 0; c < 3; ++c) r.w[k][c] = 0.0; }
        if (!FW) {
            double dq[3];
            for (int c = 0; c < M; ++c) dq[c] = qr[c] - ql[c];
            if (SYS == ADJ_SYS_AC1D) {         // acoustics_rp_1d, equations.py:125-140
                double zl = ml[1], zr = mr[1];
                double a1 = (-dq[0] + zr * dq[1]) / (zl + zr);
                double a2 = (dq[0] + zl * dq[1]) / (zl + zr);
                r.w[0][0] = -a1 * zl; r.w[0][1] = a1;
                r.w[1][0] = a2 * zr;  r.w[1][1] = a2;
                r.s[0] = -ml[0]; r.s[1] = mr[0];
            } else if (SYS == ADJ_SYS_AC2D) {  // acoustics_rp_normal_2d, equations.py:143-169
                double zl = ml[1], zr = mr[1];
                double a1 = (-dq[0] + zr * dq[mu]) / (zl + zr);
                double a2 = (dq[0] + zl * dq[mu]) / (zl + zr);
                r.w[0][0] = -a1 * zl; r.w[0][mu] = a1;
                r.w[1][mv] = dq[mv];
                r.w[2][0] = a2 * zr;  r.w[2][mu] = a2;
                r.s[0] = -ml[0]; r.s[1] = 0.0; r.s[2] = mr[0];
            } else {                           // swe_linear_rp, equations.py:198-224
                double cl = ml[0], cr = mr[0];
                double a1 = (cr * dq[0] - dq[mu]) / (cl + cr);
                double a2 = (cl * dq[0] + dq[mu]) / (cl + cr);
                r.w[0][0] = a1; r.w[0][mu] = -a1 * cl;
                r.w[1][mv] = dq[mv];
                r.w[2][0] = a2; r.w[2][mu] = a2 * cr;
                r.s[0] = -cl; r.s[1] = 0.0; r.s[2] = cr;
            }
        } else {
            // adjoint_flux + adjoint_fwave_rp, equations.py:249-320
            double fl[3] = {0.0, 0.0, 0.0}, fr[3] = {0.0, 0.0, 0.0}, df[3];
            if (SYS == ADJ_SYS_AC1D) {
                fl[0] = ql[1] / ml[2]; fl[1] = ml[3] * ql[0];
                fr[0] = qr[1] / mr[2]; fr[1] = mr[3] * qr[0];
            } else if (SYS == ADJ_SYS_AC2D) {
                fl[0] = ql[mu] / ml[2]; fl[mu] = ml[3] * ql[0];
                fr[0] = qr[mu] / mr[2]; fr[mu] = mr[3] * qr[0];
            } else {
                fl[0] = g * ml[1] * ql[mu]; fl[mu] = ql[0];
                fr[0] = g * mr[1] * qr[mu]; fr[mu] = qr[0];
            }
            for (int c = 0; c < M; ++c) df[c] = fr[c] - fl[c];
            if (SYS == ADJ_SYS_AC1D) {
                double zl = ml[1], zr = mr[1];
                double b1 = (zr * df[0] - df[1]) / (zl + zr);
                double b2 = (zl * df[0] + df[1]) / (zl + zr);
                r.w[0][0] = b1; r.w[0][1] = -b1 * zl;
                r.w[1][0] = b2; r.w[1][1] = b2 * zr;
                r.s[0] = -ml[0]; r.s[1] = mr[0];
            } else if (SYS == ADJ_SYS_AC2D) {
                double zl = ml[1], zr = mr[1];
                double b1 = (zr * df[0] - df[mu]) / (zl + zr);
                double b2 = (zl * df[0] + df[mu]) / (zl + zr);
                r.w[0][0] = b1; r.w[0][mu] = -b1 * zl;
                r.w[2][0] = b2; r.w[2][mu] = b2 * zr;
                r.s[0] = -ml[0]; r.s[1] = 0.0; r.s[2] = mr[0];
            } else {
                double cl = ml[0], cr = mr[0];
                double b1 = (cr * df[mu] - df[0]) / (cl + cr);
                double b2 = (cl * df[mu] + df[0]) / (cl + cr);
                r.w[0][0] = -b1 * cl; r.w[0][mu] = b1;
                r.w[2][0] = b2 * cr;  r.w[2][mu] = b2;
                r.s[0] = -cl; r.s[1] = 0.0; r.s[2] = cr;
            }
        }
        fluct(r);
        if (REV) {  // TimeReversed.normal_rp, equations.py:517-527
            Rp t = r;
            for (int k = 0; k < NW; ++k) {
                r.s[k] = -t.s[NW - 1 - k];
                for (int c = 0; c < 3; ++c) r.w[k][c] = FW ? -t.w[NW - 1 - k][c] : t.w[NW - 1 - k][c];
            }
            for (int c = 0; c < 3; ++c) { r.am[c] = -t.ap[c]; r.ap[c] = -t.am[c]; }
        }
    }

    // One interface solve between cells L and R along `axis` (_solve_axis).
    static __device__ K1X_FACE_INL void face(const PatchView& P, int axis, int iL, int jL,
                                             int iR, int jR, double g, Rp& r) {
        double ql[3] = {0, 0, 0}, qr[3] = {0, 0, 0};
        for (int c = 0; c < M; ++c) { ql[c] = P.Q(c, iL, jL); qr[c] = P.Q(c, iR, jR); }
        if (SWE) {
            // _swe_effective_states, solver.py:357-380
            const int mu = 1 + axis;
            double dL = P.A(1, iL, jL), dR = P.A(1, iR, jR);
            bool wl = dL > 0.0, wr = dR > 0.0, dd = !wl && !wr;
            double qle[3], qre[3];
            for (int c = 0; c < 3; ++c) {
                qle[c] = wl ? ql[c] : (c == mu ? -qr[c] : qr[c]);
                qre[c] = wr ? qr[c] : (c == mu ? -ql[c] : ql[c]);
            }
            double dl = wl ? dL : dR, dr = wr ? dR : dL;
            if (dd) { dl = 1.0; dr = 1.0; }
            double ml[4] = {sqrt(g * dl), dl, 0.0, 0.0};
            double mr[4] = {sqrt(g * dr), dr, 0.0, 0.0};
            normal(axis, qle, qre, ml, mr, g, r);
            if (dd) {  // solver.py:406-409
                for (int k = 0; k < 3; ++k) { r.s[k] = 0.0; for (int c = 0; c < 3; ++c) r.w[k][c] = 0.0; }
                for (int c = 0; c < 3; ++c) { r.am[c] = 0.0; r.ap[c] = 0.0; }
            }
        } else {
            double ml[4], mr[4];
            for (int k = 0; k < 4; ++k) { ml[k] = P.A(k, iL, jL); mr[k] = P.A(k, iR, jR); }
            normal(axis, ql, qr, ml, mr, g, r);
        }
    }

    // Transverse split (equations.py:172-191, 227-242, 323-349; TimeReversed 529-531),
    // materials of the cells below/above; SWE clamps dry cells (solver.py:383-387).
    static __device__ K1X_FACE_INL void trans(const PatchView& P, int axis, const double* f,
                                              int ib, int jb, int ia, int ja, double g,
                                              double* bm, double* bp) {
        const int mv = 2 - axis;
        double m_[3] = {0, 0, 0}, p_[3] = {0, 0, 0};
        if (SWE) {
            double db = P.A(1, ib, jb), da = P.A(1, ia, ja);
            double cb = sqrt(g * (db > 0.0 ? db : 1.0));
            double ca = sqrt(g * (da > 0.0 ? da : 1.0));
            double den = cb + ca;
            if (!FW) {
                double bd = (ca * f[0] - f[mv]) / den;
                double bu = (cb * f[0] + f[mv]) / den;
                m_[0] = -cb * bd; m_[mv] = -cb * (-bd * cb);
                p_[0] = ca * bu;  p_[mv] = ca * (bu * ca);
            } else {
                double bd = (ca * f[mv] - f[0]) / den;
                double bu = (cb * f[mv] + f[0]) / den;
                m_[0] = -cb * (-bd * cb); m_[mv] = -cb * bd;
                p_[0] = ca * (bu * ca);   p_[mv] = ca * bu;
            }
        } else {
            double cb = P.A(0, ib, jb), zb = P.A(1, ib, jb);
            double ca = P.A(0, ia, ja), za = P.A(1, ia, ja);
            if (!FW) {
                double bd = (-f[0] + za * f[mv]) / (zb + za);
                double bu = (f[0] + zb * f[mv]) / (zb + za);
                m_[0] = -cb * (-bd * zb); m_[mv] = -cb * bd;
                p_[0] = ca * (bu * za);   p_[mv] = ca * bu;
            } else {
                double bd = (za * f[0] - f[mv]) / (zb + za);
                double bu = (zb * f[0] + f[mv]) / (zb + za);
                m_[0] = -cb * bd; m_[mv] = -cb * (-bd * zb);
                p_[0] = ca * bu;  p_[mv] = ca * (bu * za);
            }
        }
        for (int c = 0; c < 3; ++c) {
            if (REV) { bm[c] = -p_[c]; bp[c] = -m_[c]; }
            else { bm[c] = m_[c]; bp[c] = p_[c]; }
        }
    }

    // _limited_waves + _correction_flux (solver.py:317-348) at face `c`
    // with upwind neighbours `u` (face - 1) and `d` (face + 1).
    static ADJ_D void corr(const Rp& c, const Rp& u, const Rp& d, double dtd, int lim, double* F) {
        double lw[3][3];
        for (int k = 0; k < NW; ++k) {
            if (lim == ADJ_LIM_NONE) {
                for (int q = 0; q < M; ++q) lw[k][q] = c.w[k][q];
            } else {
                double dots = c.w[k][0] * c.w[k][0], dup = u.w[k][0] * c.w[k][0], ddn = d.w[k][0] * c.w[k][0];
                for (int q = 1; q < M; ++q) {
                    dots = dots + c.w[k][q] * c.w[k][q];
                    dup = dup + u.w[k][q] * c.w[k][q];
                    ddn = ddn + d.w[k][q] * c.w[k][q];
                }
                double upw = c.s[k] > 0.0 ? dup : ddn;
                double th = dots > 0.0 ? upw / dots : 0.0;
                double phi = limiter_phi(lim, th);
                for (int q = 0; q < M; ++q) lw[k][q] = phi * c.w[k][q];
            }
        }
        double coef[3];
        for (int k = 0; k < NW; ++k) {
            double as = fabs(c.s[k]);
            if (FW) {
                double sg = c.s[k] > 0.0 ? 1.0 : (c.s[k] < 0.0 ? -1.0 : 0.0);
                coef[k] = (0.5 * sg) * (1.0 - dtd * as);
            } else {
                coef[k] = (0.5 * as) * (1.0 - dtd * as);
            }
        }
        for (int q = 0; q < M; ++q) {
            double s = coef[0] * lw[0][q];
            for (int k = 1; k < NW; ++k) s = s + coef[k] * lw[k][q];
            F[q] = s;
        }
    }

    static ADJ_D bool wet(const PatchView& P, int i, int j) { return P.A(1, i, j) > 0.0; }

    // ftil at x-face (i,j) after transverse terms T3/T4 and SWE face mask (solver.py:470-500).
    // XF(i, j, r) / YF(i, j, r) give the x-face (i | i+1, row j) / y-face (j | j+1,
    // column i) solve: computed on the spot, or read from a tile's shared memory.
    template <class XF, class YF>
    static __device__ K1X_TIL_INL void ftil_t(const PatchView& P, XF&& xf, YF&& yf, int i, int j, double dtdx,
                                              double dtdy, double g, int lim, double* F) {
        Rp c, u, d;
        xf(i, j, c);
        xf(i - 1, j, u);
        xf(i + 1, j, d);
        corr(c, u, d, dtdx, lim, F);
        const double h = 0.5 * dtdy;
        double bm[3], bp[3];
        Rp y;
        yf(i + 1, j, y);                                   // amdq_y(i+1, j) -> bm
        trans(P, 1, y.am, i, j, i + 2, j, g, bm, bp);
        for (int q = 0; q < 3; ++q) F[q] = F[q] - h * bm[q];
        yf(i, j, y);                                       // amdq_y(i, j) -> bp
        trans(P, 1, y.am, i - 1, j, i + 1, j, g, bm, bp);
        for (int q = 0; q < 3; ++q) F[q] = F[q] - h * bp[q];
        yf(i + 1, j - 1, y);                               // apdq_y(i+1, j-1) -> bm
        trans(P, 1, y.ap, i, j, i + 2, j, g, bm, bp);
        for (int q = 0; q < 3; ++q) F[q] = F[q] - h * bm[q];
        yf(i, j - 1, y);                                   // apdq_y(i, j-1) -> bp
        trans(P, 1, y.ap, i - 1, j, i + 1, j, g, bm, bp);
        for (int q = 0; q < 3; ++q) F[q] = F[q] - h * bp[q];
        if (SWE && !(wet(P, i, j) && wet(P, i + 1, j)))
            for (int q = 0; q < 3; ++q) F[q] = 0.0;
    }

    // gtil at y-face (i,j) after transverse terms T1/T2 and SWE face mask
    template <class XF, class YF>
    static __device__ K1X_TIL_INL void gtil_t(const PatchView& P, XF&& xf, YF&& yf, int i, int j, double dtdx,
                                              double dtdy, double g, int lim, double* G) {
        Rp c, u, d;
        yf(i, j, c);
        yf(i, j - 1, u);
        yf(i, j + 1, d);
        corr(c, u, d, dtdy, lim, G);
        const double h = 0.5 * dtdx;
        double bm[3], bp[3];
        Rp x;
        xf(i, j + 1, x);                                   // amdq_x(i, j+1) -> bm
        trans(P, 0, x.am, i, j, i, j + 2, g, bm, bp);
        for (int q = 0; q < 3; ++q) G[q] = G[q] - h * bm[q];
        xf(i, j, x);                                       // amdq_x(i, j) -> bp
        trans(P, 0, x.am, i, j - 1, i, j + 1, g, bm, bp);
        for (int q = 0; q < 3; ++q) G[q] = G[q] - h * bp[q];
        xf(i - 1, j + 1, x);                               // apdq_x(i-1, j+1) -> bm
        trans(P, 0, x.ap, i, j, i, j + 2, g, bm, bp);
        for (int q = 0; q < 3; ++q) G[q] = G[q] - h * bm[q];
        xf(i - 1, j, x);                                   // apdq_x(i-1, j) -> bp
        trans(P, 0, x.ap, i, j - 1, i, j + 1, g, bm, bp);
        for (int q = 0; q < 3; ++q) G[q] = G[q] - h * bp[q];
        if (SWE && !(wet(P, i, j) && wet(P, i, j + 1)))
            for (int q = 0; q < 3; ++q) G[q] = 0.0;
    }

    static __device__ K1X_TIL_INL void ftil(const PatchView& P, int i, int j, double dtdx, double dtdy, double g,
                                            int lim, double* F) {
        ftil_t(P, [&](int a, int b, Rp& r) { face(P, 0, a, b, a + 1, b, g, r); },
               [&](int a, int b, Rp& r) { face(P, 1, a, b, a, b + 1, g, r); }, i, j, dtdx, dtdy, g, lim, F);
    }

    static __device__ K1X_TIL_INL void gtil(const PatchView& P, int i, int j, double dtdx, double dtdy, double g,
                                            int lim, double* G) {
        gtil_t(P, [&](int a, int b, Rp& r) { face(P, 0, a, b, a + 1, b, g, r); },
               [&](int a, int b, Rp& r) { face(P, 1, a, b, a, b + 1, g, r); }, i, j, dtdx, dtdy, g, lim, G);
    }
};

template <int SYS, int FORM, bool REV>
__global__ void __launch_bounds__(256) k1_exact(AdjStepArgs a) {
    using S = Step<SYS, FORM, REV>;
    constexpr int M = S::M;
    const AdjTile t = a.tiles[blockIdx.x];
    if (a.ndim == 2 ? (t.ni > 16 || t.nj > 16) : t.ni > 256) {   // not the adj_step_tile_shape the
        if (threadIdx.x == 0) a.nonfinite[t.patch] = 2;          // CTA covers: reported, nothing written
        return;
    }
    const AdjPatch p = a.patches[t.patch];
    const int g = a.ghost;
    int di, dj;
    if (a.ndim == 2) { di = threadIdx.x >> 4; dj = threadIdx.x & 15; }
    else { di = threadIdx.x; dj = 0; }
    const bool active = di < t.ni && dj < t.nj;
    PatchView P{a.q_in + p.offset, a.aux + p.offset, a.comp_stride, a.aux_stride, p.pitch};
    double smx = 0.0, smy = 0.0;
    bool bad = false;
    if (active) {
        const int i = g + t.i0 + di;
        const double dtdx = a.dtdx, dtdy = a.dtdy, gr = a.gravity;
        double dq[3] = {0.0, 0.0, 0.0};
        double qn[3];
        if (SYS == ADJ_SYS_AC1D) {
            Rp l, r, ll, rr;
            S::face(P, 0, i - 1, 0, i, 0, gr, l);
            S::face(P, 0, i, 0, i + 1, 0, gr, r);
            S::face(P, 0, i - 2, 0, i - 1, 0, gr, ll);
            S::face(P, 0, i + 1, 0, i + 2, 0, gr, rr);
            double Fr[3], Fl[3];
            S::corr(r, l, rr, dtdx, a.limiter, Fr);
            S::corr(l, ll, r, dtdx, a.limiter, Fl);
            for (int c = 0; c < M; ++c) {
                dq[c] = dq[c] - dtdx * l.ap[c];
                dq[c] = dq[c] - dtdx * r.am[c];
                dq[c] = dq[c] - dtdx * (Fr[c] - Fl[c]);
            }
            for (int k = 0; k < S::NW; ++k) smx = fmax(smx, fabs(l.s[k]));
            if (i == g + p.nx - 1) for (int k = 0; k < S::NW; ++k) smx = fmax(smx, fabs(r.s[k]));
            for (int c = 0; c < M; ++c) qn[c] = P.Q(c, i, 0) + dq[c];
            for (int c = 0; c < M; ++c) {
                a.q_out[c * a.comp_stride + p.offset + i] = qn[c];
                bad |= !isfinite(qn[c]);
            }
        } else {
            const int j = g + t.j0 + dj;
            {
                Rp f;
                S::face(P, 0, i - 1, j, i, j, gr, f);
                for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdx * f.ap[c];
                for (int k = 0; k < 3; ++k) smx = fmax(smx, fabs(f.s[k]));
                S::face(P, 0, i, j, i + 1, j, gr, f);
                for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdx * f.am[c];
                if (i == g + p.nx - 1) for (int k = 0; k < 3; ++k) smx = fmax(smx, fabs(f.s[k]));
                S::face(P, 1, i, j - 1, i, j, gr, f);
                for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdy * f.ap[c];
                for (int k = 0; k < 3; ++k) smy = fmax(smy, fabs(f.s[k]));
                S::face(P, 1, i, j, i, j + 1, gr, f);
                for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdy * f.am[c];
                if (j == g + p.ny - 1) for (int k = 0; k < 3; ++k) smy = fmax(smy, fabs(f.s[k]));
            }
            double Fr[3], Fl[3];
            S::ftil(P, i, j, dtdx, dtdy, gr, a.limiter, Fr);
            S::ftil(P, i - 1, j, dtdx, dtdy, gr, a.limiter, Fl);
            for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdx * (Fr[c] - Fl[c]);
            S::gtil(P, i, j, dtdx, dtdy, gr, a.limiter, Fr);
            S::gtil(P, i, j - 1, dtdx, dtdy, gr, a.limiter, Fl);
            for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdy * (Fr[c] - Fl[c]);
            if (S::SWE) {
                double w = S::wet(P, i, j) ? 1.0 : 0.0;
                for (int c = 0; c < 3; ++c) dq[c] = dq[c] * w;
            }
            for (int c = 0; c < 3; ++c) qn[c] = P.Q(c, i, j) + dq[c];
            const int64_t o = p.offset + (int64_t)i * p.pitch + j;
            for (int c = 0; c < 3; ++c) {
                a.q_out[c * a.comp_stride + o] = qn[c];
                bad |= !isfinite(qn[c]);
            }
        }
    }
    smx = warp_max(smx);
    smy = warp_max(smy);
    unsigned anybad = __ballot_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        if (smx > 0.0) atomic_max_nonneg(&a.speed_max[2 * t.patch], smx);
        if (smy > 0.0) atomic_max_nonneg(&a.speed_max[2 * t.patch + 1], smy);
        if (anybad) a.nonfinite[t.patch] = 1;
    }
}

// 2D, tiled: a CTA owns a 16x16 AdjTile.  Every interface solve its stencil
// needs is computed once into shared memory (phase 0), then every ftil /
// gtil of the tile's faces (phase 1), then the cell updates (phase 2) -- the
// per-cell kernel above recomputes ~32 interface solves and 4 ftil/gtil per
// cell.  Same functions, same operands, same accumulation order: bitwise
// equal to k1_exact.
constexpr int XT = 16;
constexpr int XS_N = (XT + 3) * (XT + 2);     // x-faces: i in [bi0-2, bi0+ni], j in [bj0-1, bj0+nj]
constexpr int YS_N = (XT + 2) * (XT + 3);     // y-faces: i in [bi0-1, bi0+ni], j in [bj0-2, bj0+nj]
constexpr int TILED_SMEM = (XS_N + YS_N) * (int)sizeof(Rp) + 2 * (XT + 1) * XT * 3 * (int)sizeof(double);

template <int SYS, int FORM, bool REV>
__global__ void __launch_bounds__(256) k1_exact_tiled(AdjStepArgs a) {
    using S = Step<SYS, FORM, REV>;
    extern __shared__ __align__(16) unsigned char smem_t[];
    Rp* XS = reinterpret_cast<Rp*>(smem_t);
    Rp* YS = XS + XS_N;
    double* FS = reinterpret_cast<double*>(YS + YS_N);   // ftil, face i = bi0-1+a, row bj0+b: [(a*XT+b)*3]
    double* GS = FS + (XT + 1) * XT * 3;                  // gtil, column bi0+a, face j = bj0-1+b: [(a*(XT+1)+b)*3]
    const AdjTile t = a.tiles[blockIdx.x];
    if (t.ni > XT || t.nj > XT) {   // the shared-memory face tables hold at most XT x XT cells
        if (threadIdx.x == 0) a.nonfinite[t.patch] = 2;
        return;
    }
    const AdjPatch p = a.patches[t.patch];
    const int g = a.ghost;
    const int ni = t.ni, nj = t.nj, bi0 = g + t.i0, bj0 = g + t.j0;
    const int nxj = nj + 2, nyj = nj + 3;
    PatchView P{a.q_in + p.offset, a.aux + p.offset, a.comp_stride, a.aux_stride, p.pitch};
    const double dtdx = a.dtdx, dtdy = a.dtdy, gr = a.gravity;
    for (int k = threadIdx.x; k < (ni + 3) * nxj; k += blockDim.x) {
        const int i = bi0 - 2 + k / nxj, j = bj0 - 1 + k % nxj;
        S::face(P, 0, i, j, i + 1, j, gr, XS[k]);
    }
    for (int k = threadIdx.x; k < (ni + 2) * nyj; k += blockDim.x) {
        const int i = bi0 - 1 + k / nyj, j = bj0 - 2 + k % nyj;
        S::face(P, 1, i, j, i, j + 1, gr, YS[k]);
    }
    __syncthreads();
    auto xf = [&](int i, int j, Rp& r) { r = XS[(i - (bi0 - 2)) * nxj + (j - (bj0 - 1))]; };
    auto yf = [&](int i, int j, Rp& r) { r = YS[(i - (bi0 - 1)) * nyj + (j - (bj0 - 2))]; };
    for (int k = threadIdx.x; k < (ni + 1) * nj; k += blockDim.x) {
        const int ai = k / nj, bj = k % nj;
        S::ftil_t(P, xf, yf, bi0 - 1 + ai, bj0 + bj, dtdx, dtdy, gr, a.limiter, FS + (ai * XT + bj) * 3);
    }
    for (int k = threadIdx.x; k < ni * (nj + 1); k += blockDim.x) {
        const int ai = k / (nj + 1), bj = k % (nj + 1);
        S::gtil_t(P, xf, yf, bi0 + ai, bj0 - 1 + bj, dtdx, dtdy, gr, a.limiter, GS + (ai * (XT + 1) + bj) * 3);
    }
    __syncthreads();
    const int di = threadIdx.x >> 4, dj = threadIdx.x & 15;
    double smx = 0.0, smy = 0.0;
    bool bad = false;
    if (di < ni && dj < nj) {
        const int i = bi0 + di, j = bj0 + dj;
        double dq[3] = {0.0, 0.0, 0.0};
        Rp f;
        xf(i - 1, j, f);
        for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdx * f.ap[c];
        for (int k = 0; k < 3; ++k) smx = fmax(smx, fabs(f.s[k]));
        xf(i, j, f);
        for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdx * f.am[c];
        if (i == g + p.nx - 1) for (int k = 0; k < 3; ++k) smx = fmax(smx, fabs(f.s[k]));
        yf(i, j - 1, f);
        for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdy * f.ap[c];
        for (int k = 0; k < 3; ++k) smy = fmax(smy, fabs(f.s[k]));
        yf(i, j, f);
        for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdy * f.am[c];
        if (j == g + p.ny - 1) for (int k = 0; k < 3; ++k) smy = fmax(smy, fabs(f.s[k]));
        const double* Fr = FS + ((di + 1) * XT + dj) * 3;
        const double* Fl = FS + (di * XT + dj) * 3;
        for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdx * (Fr[c] - Fl[c]);
        const double* Gr = GS + (di * (XT + 1) + dj + 1) * 3;
        const double* Gl = GS + (di * (XT + 1) + dj) * 3;
        for (int c = 0; c < 3; ++c) dq[c] = dq[c] - dtdy * (Gr[c] - Gl[c]);
        if (S::SWE) {
            double w = S::wet(P, i, j) ? 1.0 : 0.0;
            for (int c = 0; c < 3; ++c) dq[c] = dq[c] * w;
        }
        const int64_t o = p.offset + (int64_t)i * p.pitch + j;
        for (int c = 0; c < 3; ++c) {
            const double qn = P.Q(c, i, j) + dq[c];
            a.q_out[c * a.comp_stride + o] = qn;
            bad |= !isfinite(qn);
        }
    }
    smx = warp_max(smx);
    smy = warp_max(smy);
    unsigned anybad = __ballot_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        if (smx > 0.0) atomic_max_nonneg(&a.speed_max[2 * t.patch], smx);
        if (smy > 0.0) atomic_max_nonneg(&a.speed_max[2 * t.patch + 1], smy);
        if (anybad) a.nonfinite[t.patch] = 1;
    }
}

#ifndef K1X_TILED
#define K1X_TILED 1
#endif

template <int SYS, int FORM, bool REV>
static int launch(const AdjStepArgs& a, cudaStream_t st) {
    if (K1X_TILED && a.ndim == 2 && SYS != ADJ_SYS_AC1D) {
        // opt-in shared memory is a per-device function attribute: set once per device
        static unsigned long long attr_set = 0ull;
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return check_launch("k1_exact_tiled");
        if (!(attr_set & (1ull << dev))) {
            if (cudaFuncSetAttribute(k1_exact_tiled<SYS, FORM, REV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     TILED_SMEM) != cudaSuccess)
                return check_launch("k1_exact_tiled (shared memory attribute)");
            attr_set |= 1ull << dev;
        }
        k1_exact_tiled<SYS, FORM, REV><<<a.ntile, 256, TILED_SMEM, st>>>(a);
        return ADJ_OK;
    }
    k1_exact<SYS, FORM, REV><<<a.ntile, 256, 0, st>>>(a);
    return ADJ_OK;
}

template <int SYS>
static int dispatch_form(const AdjStepArgs& a, cudaStream_t st) {
    if (a.form == ADJ_FORM_WAVE)
        return a.reversed ? launch<SYS, ADJ_FORM_WAVE, true>(a, st) : launch<SYS, ADJ_FORM_WAVE, false>(a, st);
    return a.reversed ? launch<SYS, ADJ_FORM_FWAVE, true>(a, st) : launch<SYS, ADJ_FORM_FWAVE, false>(a, st);
}

}  // namespace exact

int step_exact(const AdjStepArgs& a, cudaStream_t st) {
    if (a.ntile <= 0) return ADJ_OK;
    int rc;
    switch (a.system) {
        case ADJ_SYS_AC1D: rc = exact::dispatch_form<ADJ_SYS_AC1D>(a, st); break;
        case ADJ_SYS_AC2D: rc = exact::dispatch_form<ADJ_SYS_AC2D>(a, st); break;
        case ADJ_SYS_SWE2D: rc = exact::dispatch_form<ADJ_SYS_SWE2D>(a, st); break;
        default: return ADJ_ERR_BAD_ARG;
    }
    if (rc != ADJ_OK) return rc;
    return check_launch("k1_exact");
}

}  // namespace adj
