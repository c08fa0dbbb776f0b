// K1, FAST variant (2D): warp-strip register-marching wave-propagation step.
//
// Work unit: one warp per AdjTile = an output strip of nj <= 28 rows (y, the
// contiguous axis) by ni columns (x).  Lane l owns row j0-2+l for the whole
// strip, so every global load/store is a coalesced 32-lane row segment; the
// warp marches along x keeping the last three columns, the last three
// x-faces and the pipeline values in registers.  y-neighbour data moves
// between lanes with warp shuffles; no shared memory, no recomputation along
// x, 4/32 halo lanes along y.
//
// Algebra (same scheme as the reference, reorganised; agrees with the EXACT
// variant / the numpy reference to ~1e-16 norm-relative per step):
//  * every 2D system in both forms has waves in components (0, mu) only, with
//    eigenvectors (±m, 1) or (1, ±m) (m = impedance z or speed c), so a wave
//    is a scalar strength sigma times a material vector;
//  * the limiter phi(theta)*W with theta = (W_up.W)/(W.W) is evaluated
//    division-free as lim(A, B) / (1 + m^2) with A = sigma (1+m^2) and
//    B = sigma_up (1 + m m_up) (identical for minmod / MC / superbee);
//  * the two transverse splits feeding a cell use the same pair of
//    materials, so the entering fluctuations are summed before splitting;
//  * material-only reciprocals use rcp.approx + two Newton steps.
// Reference: step_patch_2d solver.py:442-512, equations.py:143-349,
// _limited_waves / _correction_flux solver.py:317-348, TimeReversed
// equations.py:496-534.  Levels with dry shallow-water cells use the EXACT
// variant (host dispatch), so no wet/dry logic is needed here.
#include "adj_common.cuh"

namespace adj {

void fast_tile_shape(int ndim, int32_t* ni, int32_t* nj) {
    if (ndim == 2) { *ni = 128; *nj = 28; } else { *ni = 256; *nj = 1; }
}

namespace fast {

constexpr unsigned FULL = 0xffffffffu;

ADJ_D double rcp(double x) {  // x > 0, normal
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

ADJ_D double sh_dn(double v) { return __shfl_down_sync(FULL, v, 1); }  // from lane+1 (row j+1)
ADJ_D double sh_up(double v) { return __shfl_up_sync(FULL, v, 1); }    // from lane-1 (row j-1)

// division-free limited strength lim(A,B) = phi(B/A) * A (solver.py:65-77)
template <int LIM>
ADJ_D double limab(double A, double B) {
    const double a = fabs(A);
    const double b = A < 0.0 ? -B : B;
    double r;
    if (LIM == ADJ_LIM_MINMOD) r = fmax(0.0, fmin(a, b));
    else if (LIM == ADJ_LIM_MC) r = fmax(0.0, fmin(fmin(0.5 * (a + b), a + a), b + b));
    else r = fmax(0.0, fmax(fmin(a, b + b), fmin(a + a, b)));  // superbee
    return copysign(r, A);
}

// Per-cell material quantities.  m: eigen material (z for acoustics, c for
// shallow water); k1i = 1/(1+m^2); kx, ky: correction magnitudes
// (wave: 0.5 c (1 - dtd c); f-wave: 0.5 (1 - dtd c)); tr: transverse helper
// (acoustics K = c z, shallow water c^2); fx: f-wave flux factor (acoustics
// 1/rho, shallow water g h = c^2).
struct Mat {
    double c, m, k1i, kx, ky, tr, fx;
};

template <int SYS, int FORM>
ADJ_D Mat make_mat(double c, double z, double dtdx, double dtdy) {
    constexpr bool SWE = SYS == ADJ_SYS_SWE2D, FW = FORM == ADJ_FORM_FWAVE;
    Mat t;
    t.c = c;
    t.m = SWE ? c : z;
    t.k1i = rcp(fma(t.m, t.m, 1.0));
    const double hx = 0.5 * fma(-dtdx, c, 1.0), hy = 0.5 * fma(-dtdy, c, 1.0);
    t.kx = FW ? hx : c * hx;
    t.ky = FW ? hy : c * hy;
    t.tr = SWE ? c * c : c * z;
    t.fx = FW ? (SWE ? c * c : c / z) : 0.0;
    return t;
}

// One face: strengths of the two non-trivial families in reference order
// (family 0 left-going with left material, family 1 right-going), the
// fluctuations (component 0, component mu) and P = 1 + mL mR.
struct Face {
    double s0, s1, P;
    double am0, am1, ap0, ap1;   // (component 0, normal component)
};

template <int SYS, int FORM, bool REV>
ADJ_D Face solve_face(double qL0, double qLn, double qR0, double qRn, const Mat& L, const Mat& R) {
    constexpr bool SWE = SYS == ADJ_SYS_SWE2D, FW = FORM == ADJ_FORM_FWAVE;
    Face f;
    const double inv = rcp(L.m + R.m);
    if (!FW) {
        const double d0 = qR0 - qL0, dn = qRn - qLn;
        if (!SWE) {       // acoustics_rp_normal_2d
            f.s0 = (R.m * dn - d0) * inv;
            f.s1 = (L.m * dn + d0) * inv;
            // amdq = -cL W1 = s0 (cL zL, -cL) ; apdq = cR W2 = s1 (cR zR, cR)
            f.am0 = f.s0 * L.tr; f.am1 = -f.s0 * L.c;
            f.ap0 = f.s1 * R.tr; f.ap1 = f.s1 * R.c;
        } else {          // swe_linear_rp
            f.s0 = (R.c * d0 - dn) * inv;
            f.s1 = (L.c * d0 + dn) * inv;
            f.am0 = -f.s0 * L.c; f.am1 = f.s0 * L.tr;
            f.ap0 = f.s1 * R.c;  f.ap1 = f.s1 * R.tr;
        }
    } else {              // adjoint_fwave_rp
        double d0, dn;
        if (!SWE) { d0 = qRn * R.fx - qLn * L.fx; dn = R.tr * qR0 - L.tr * qL0; }   // q_mu/rho, K q0
        else { d0 = R.fx * qRn - L.fx * qLn; dn = qR0 - qL0; }
        if (!SWE) {
            f.s0 = (R.m * d0 - dn) * inv;
            f.s1 = (L.m * d0 + dn) * inv;
            f.am0 = f.s0; f.am1 = -f.s0 * L.m;
            f.ap0 = f.s1; f.ap1 = f.s1 * R.m;
        } else {
            f.s0 = (R.c * dn - d0) * inv;
            f.s1 = (L.c * dn + d0) * inv;
            f.am0 = -f.s0 * L.c; f.am1 = f.s0;
            f.ap0 = f.s1 * R.c;  f.ap1 = f.s1;
        }
    }
    if (REV) {  // TimeReversed: amdq' = -apdq, apdq' = -amdq
        double a0 = f.am0, a1 = f.am1;
        f.am0 = -f.ap0; f.am1 = -f.ap1;
        f.ap0 = -a0; f.ap1 = -a1;
    }
    f.P = fma(L.m, R.m, 1.0);
    return f;
}

// Limited correction flux (component 0, normal component) of face f.
//   non-reversed: family 0 upwind = next face, family 1 upwind = previous face
//   reversed:     family 0 upwind = previous face, family 1 upwind = next face
template <int SYS, int FORM, bool REV, int LIM>
ADJ_D void correction(const Face& f, double s0_nb, double P0_nb, double s1_nb, double P1_nb,
                      const Mat& L, const Mat& R, double kL, double kR, double& F0, double& Fn) {
    constexpr bool SWE = SYS == ADJ_SYS_SWE2D, FW = FORM == ADJ_FORM_FWAVE;
    constexpr bool MPOS0 = (!SWE && !FW) || (SWE && FW);  // material multiplies component 0
    double p0, p1;
    if (LIM == ADJ_LIM_NONE) {
        p0 = f.s0; p1 = f.s1;
    } else {
        const double A0 = f.s0 * fma(L.m, L.m, 1.0);
        const double A1 = f.s1 * fma(R.m, R.m, 1.0);
        const double B0 = s0_nb * (REV ? P0_nb : f.P);
        const double B1 = s1_nb * (REV ? P1_nb : f.P);
        p0 = limab<LIM>(A0, B0) * L.k1i;
        p1 = limab<LIM>(A1, B1) * R.k1i;
    }
    // coefficients: wave 0.5|s|(1-dtd|s|) for both; f-wave sign(s) 0.5(1-dtd|s|)
    const double u0 = (FW ? -kL : kL) * p0;
    const double u1 = kR * p1;
    if (MPOS0) { F0 = (SWE ? R.c * u1 - L.c * u0 : R.m * u1 - L.m * u0); Fn = u0 + u1; }
    else { F0 = u0 + u1; Fn = (SWE ? R.c * u1 - L.c * u0 : R.m * u1 - L.m * u0); }
}

// Transverse split of an entering fluctuation (component 0 = f0; its
// transverse component is zero for every 2D system here), scaled by h.
// Returns bm (to the lower transverse face) and bp (upper), components
// (0, transverse velocity).
template <int SYS, int FORM, bool REV>
ADJ_D void transverse(double f0, double h, const Mat& b, const Mat& a,
                      double& bm0, double& bmv, double& bp0, double& bpv) {
    constexpr bool SWE = SYS == ADJ_SYS_SWE2D, FW = FORM == ADJ_FORM_FWAVE;
    const double t = (h * f0) * rcp(b.m + a.m);
    double m0, mv, p0, pv;
    if (!FW) {
        if (!SWE) { m0 = -b.tr * t; mv = b.c * t; p0 = a.tr * t; pv = a.c * t; }
        else { const double u = (b.c * a.c) * t; m0 = -u; mv = b.c * u; p0 = u; pv = a.c * u; }
    } else {
        if (!SWE) { const double ta = a.m * t, tb = b.m * t; m0 = -b.c * ta; mv = b.tr * ta; p0 = a.c * tb; pv = a.tr * tb; }
        else { m0 = -b.tr * t; mv = b.c * t; p0 = a.tr * t; pv = a.c * t; }
    }
    if (REV) { bm0 = -p0; bmv = -pv; bp0 = -m0; bpv = -mv; }
    else { bm0 = m0; bmv = mv; bp0 = p0; bpv = pv; }
}

struct Raw { double q0, q1, q2, c, z; };

template <int SYS, int FORM, bool REV, int LIM>
__global__ void __launch_bounds__(128) k1_fast(AdjStepArgs a) {
    constexpr bool SWE = SYS == ADJ_SYS_SWE2D;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tid = blockIdx.x * 4 + warp;
    if (tid >= a.ntile) return;
    const AdjTile T = a.tiles[tid];
    const AdjPatch p = a.patches[T.patch];
    const int g = a.ghost;
    const int NY = p.ny + 2 * g;
    const int jj = g + T.j0 - 2 + lane;                       // ghost-inclusive row of this lane
    const int jl = jj < 0 ? 0 : (jj > NY - 1 ? NY - 1 : jj);  // clamped load row
    const bool out_lane = lane >= 2 && lane < 2 + T.nj;
    const bool yface_cfl = lane >= 1 && lane < 2 + T.nj;      // own top face in CFL range
    const int64_t cs = a.comp_stride, as = a.aux_stride;
    const double* __restrict__ qin = a.q_in + p.offset + jl;
    const double* __restrict__ aux = a.aux + p.offset + jl;
    double* __restrict__ qout = a.q_out + p.offset + jl;
    const int pitch = p.pitch;
    const double dtdx = a.dtdx, dtdy = a.dtdy;
    const double hx = 0.5 * dtdx, hy = 0.5 * dtdy;

    auto load = [&](int s) {
        const int64_t o = (int64_t)(g + s) * pitch;
        Raw r;
        r.q0 = __ldg(qin + o); r.q1 = __ldg(qin + cs + o); r.q2 = __ldg(qin + 2 * cs + o);
        r.c = __ldg(aux + o);
        r.z = SWE ? 0.0 : __ldg(aux + as + o);
        return r;
    };

    const int s_first = T.i0 - 2, s_last = T.i0 + T.ni + 1;
    Raw pf0 = load(s_first), pf1 = load(s_first + 1);

    // pipeline state (see header comment for the schedule)
    Mat mprv{}, mpp{};                 // materials of columns s-1, s-2
    double qprv0 = 0, qprv1 = 0, qprv2 = 0, qpp0 = 0, qpp1 = 0, qpp2 = 0;
    double cup_prv = 0, mup_prv = 0;   // row j+1 material of column s-1
    Face xp{}, xpp{};                  // x-faces s-3/2, s-5/2 (s-1/2 is computed per step)
    double corry_prv0 = 0, corry_prv2 = 0;   // corr_y of column s-1
    double bpY_prv0 = 0, bpY_prv1 = 0;       // bp of transverse(Sy(s-2))
    double ftil_old0 = 0, ftil_old1 = 0;     // ftil at face s-5/2
    double gt_pp0 = 0, gt_pp2 = 0;           // gtil of column s-2 (own top face)
    double sx_pp0 = 0, sx_pp1 = 0;           // Sx(s-2)
    double sy_prv0 = 0, sy_prv2 = 0, sy_pp0 = 0, sy_pp2 = 0;
    double smx = 0.0, smy = 0.0;
    bool bad = false;

    for (int s = s_first; s <= s_last; ++s) {
        const Raw cr = pf0;
        pf0 = pf1;
        if (s + 2 <= s_last) pf1 = load(s + 2);
        const Mat mc = make_mat<SYS, FORM>(cr.c, cr.z, dtdx, dtdy);

        // ---- B: x-face s-1/2 between columns s-1 and s
        const Face xf = solve_face<SYS, FORM, REV>(qprv0, qprv1, cr.q0, cr.q1, mprv, mc);
        if (s >= T.i0 && s <= T.i0 + T.ni && out_lane) smx = fmax(smx, fmax(mprv.c, mc.c));

        // ---- C: y-face between rows j and j+1 at column s
        const double uq0 = sh_dn(cr.q0), uq2 = sh_dn(cr.q2);
        Mat mu;
        mu.c = sh_dn(mc.c);
        mu.m = SWE ? mu.c : sh_dn(mc.m);
        mu.k1i = sh_dn(mc.k1i);
        mu.ky = sh_dn(mc.ky);
        mu.kx = 0.0;
        mu.tr = SWE ? mu.c * mu.c : mu.c * mu.m;
        mu.fx = FORM == ADJ_FORM_FWAVE ? sh_dn(mc.fx) : 0.0;
        const Face yf = solve_face<SYS, FORM, REV>(cr.q0, cr.q2, uq0, uq2, mc, mu);
        if (s >= T.i0 && s < T.i0 + T.ni && yface_cfl) smy = fmax(smy, fmax(mc.c, mu.c));
        double gc0, gc2;
        {
            // neighbours: next face = lane+1, previous face = lane-1
            const double s0n = REV ? sh_up(yf.s0) : sh_dn(yf.s0);
            const double s1n = REV ? sh_dn(yf.s1) : sh_up(yf.s1);
            const double P0n = REV ? sh_up(yf.P) : 0.0;
            const double P1n = REV ? sh_dn(yf.P) : 0.0;
            correction<SYS, FORM, REV, LIM>(yf, s0n, P0n, s1n, P1n, mc, mu, mc.ky, mu.ky, gc0, gc2);
        }
        const double apb0 = sh_up(yf.ap0), apb2 = sh_up(yf.ap1);
        const double sy0 = yf.am0 + apb0, sy2 = yf.am1 + apb2;   // Sy(s)

        // ---- D: Sx(s-1) and its transverse split with rows j-1, j+1 of column s-1
        const double sx0 = xp.ap0 + xf.am0, sx1 = xp.ap1 + xf.am1;
        double gt0, gt2;   // gtil of column s-1, own top face
        {
            Mat mb;  // row j-1 at column s-1
            mb.c = sh_up(mprv.c);
            mb.m = SWE ? mb.c : sh_up(mprv.m);
            mb.tr = SWE ? mb.c * mb.c : mb.c * mb.m;
            Mat ma;  // row j+1 at column s-1
            ma.c = cup_prv; ma.m = mup_prv;
            ma.tr = SWE ? ma.c * ma.c : ma.c * ma.m;
            double bm0, bmv, bp0, bpv;
            transverse<SYS, FORM, REV>(sx0, hx, mb, ma, bm0, bmv, bp0, bpv);
            const double bmu0 = sh_dn(bm0), bmu2 = sh_dn(bmv);   // bm of row j+1 -> own top face
            gt0 = corry_prv0 - (bp0 + bmu0);
            gt2 = corry_prv2 - (bpv + bmu2);
        }

        // ---- E: transverse of Sy(s-1) with columns s-2, s; x-limiter of face s-3/2
        double ft0, ft1;   // ftil at face s-3/2
        {
            double bm0, bmv, bp0, bpv;
            transverse<SYS, FORM, REV>(sy_prv0, hy, mpp, mc, bm0, bmv, bp0, bpv);
            double fc0, fc1;
            correction<SYS, FORM, REV, LIM>(xp, REV ? xpp.s0 : xf.s0, xpp.P, REV ? xf.s1 : xpp.s1, xf.P,
                                            mpp, mprv, mpp.kx, mprv.kx, fc0, fc1);
            ft0 = fc0 - (bpY_prv0 + bm0);
            ft1 = fc1 - (bpY_prv1 + bmv);
            bpY_prv0 = bp0; bpY_prv1 = bpv;
        }

        // ---- F: update cell s-2
        {
            const double gb0 = sh_up(gt_pp0), gb2 = sh_up(gt_pp2);
            if (s >= T.i0 + 2 && out_lane) {
                const double d0 = -dtdx * ((sx_pp0 + ft0) - ftil_old0) - dtdy * ((sy_pp0 + gt_pp0) - gb0);
                const double d1 = -dtdx * ((sx_pp1 + ft1) - ftil_old1);
                const double d2 = -dtdy * ((sy_pp2 + gt_pp2) - gb2);
                const double n0 = qpp0 + d0, n1 = qpp1 + d1, n2 = qpp2 + d2;
                const int64_t o = (int64_t)(g + s - 2) * pitch;
                qout[o] = n0; qout[cs + o] = n1; qout[2 * cs + o] = n2;
                bad |= !(isfinite(n0) && isfinite(n1) && isfinite(n2));
            }
        }

        // ---- shift the pipeline
        ftil_old0 = ft0; ftil_old1 = ft1;
        gt_pp0 = gt0; gt_pp2 = gt2;
        sx_pp0 = sx0; sx_pp1 = sx1;
        sy_pp0 = sy_prv0; sy_pp2 = sy_prv2;
        sy_prv0 = sy0; sy_prv2 = sy2;
        corry_prv0 = gc0; corry_prv2 = gc2;
        xpp = xp; xp = xf;
        mpp = mprv; mprv = mc;
        qpp0 = qprv0; qpp1 = qprv1; qpp2 = qprv2;
        qprv0 = cr.q0; qprv1 = cr.q1; qprv2 = cr.q2;
        cup_prv = mu.c; mup_prv = mu.m;
    }

    smx = warp_max(smx);
    smy = warp_max(smy);
    const unsigned anybad = __ballot_sync(FULL, bad);
    if (lane == 0) {
        if (smx > 0.0) atomic_max_nonneg(&a.speed_max[2 * T.patch], smx);
        if (smy > 0.0) atomic_max_nonneg(&a.speed_max[2 * T.patch + 1], smy);
        if (anybad) a.nonfinite[T.patch] = 1;
    }
}

template <int SYS, int FORM, bool REV>
static void launch_lim(const AdjStepArgs& a, cudaStream_t st) {
    const int blocks = (a.ntile + 3) / 4;
    switch (a.limiter) {
        case ADJ_LIM_NONE: k1_fast<SYS, FORM, REV, ADJ_LIM_NONE><<<blocks, 128, 0, st>>>(a); break;
        case ADJ_LIM_MINMOD: k1_fast<SYS, FORM, REV, ADJ_LIM_MINMOD><<<blocks, 128, 0, st>>>(a); break;
        case ADJ_LIM_MC: k1_fast<SYS, FORM, REV, ADJ_LIM_MC><<<blocks, 128, 0, st>>>(a); break;
        default: k1_fast<SYS, FORM, REV, ADJ_LIM_SUPERBEE><<<blocks, 128, 0, st>>>(a); break;
    }
}

template <int SYS>
static void launch_sys(const AdjStepArgs& a, cudaStream_t st) {
    if (a.form == ADJ_FORM_WAVE) {
        if (a.reversed) launch_lim<SYS, ADJ_FORM_WAVE, true>(a, st); else launch_lim<SYS, ADJ_FORM_WAVE, false>(a, st);
    } else {
        if (a.reversed) launch_lim<SYS, ADJ_FORM_FWAVE, true>(a, st); else launch_lim<SYS, ADJ_FORM_FWAVE, false>(a, st);
    }
}

}  // namespace fast

int step_exact(const AdjStepArgs& a, cudaStream_t st);

int step_fast(const AdjStepArgs& a, cudaStream_t st) {
    if (a.ntile <= 0) return ADJ_OK;
    if (a.ndim == 1) return step_exact(a, st);   // 1D runs the exact kernel (tile shape 256x1)
    if (a.system == ADJ_SYS_AC2D) fast::launch_sys<ADJ_SYS_AC2D>(a, st);
    else if (a.system == ADJ_SYS_SWE2D) fast::launch_sys<ADJ_SYS_SWE2D>(a, st);
    else return ADJ_ERR_BAD_ARG;
    return check_launch("k1_fast");
}

}  // namespace adj
