// K1, FAST variant (2D): warp-strip register-marching wave-propagation step.
//
// Work unit: one warp per AdjTile = an output strip of nj <= 28 rows (y, the
// contiguous axis) by ni columns (x).  Lane l owns row j0-2+l for the whole
// strip, so every global load/store is a coalesced 32-lane row segment; the
// warp marches along x keeping the last three columns, the last three
// x-faces and the pipeline values in registers.  Columns stream in through a
// per-warp cp.async ring in shared memory (6 columns ahead); y-neighbour data
// moves between lanes with warp shuffles; nothing is recomputed along x and
// 4/32 lanes are y halo.  Short strips of several patches share a warp job
// (job_offsets); persistent CTAs pull jobs from a global queue.
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
//  * material-only reciprocals use rcp.approx + one cubic Newton step.
// Instantiations: CFL (per-face speed maximum) or the static material bound;
// RST (restriction into the coarser level fused into the step); PFILL
// (ADJ_STEP_PHYS_IN: the physical ghost fill of the input inside the launch);
// SQ (dt/dx == dt/dy); WD (ADJ_STEP_WET_DRY: shallow water with dry cells,
// with per-job classes); HM (ADJ_STEP_UNIFORM_MAT: constant or per-job
// constant acoustic material, the material terms as loop invariants).
// Reference: step_patch_2d solver.py:442-512, equations.py:143-349,
// _limited_waves / _correction_flux solver.py:317-348, _swe_effective_states
// solver.py:357-387, TimeReversed equations.py:496-534.
#include "adj_common.cuh"

#ifndef K1_MIN_BLOCKS
#define K1_MIN_BLOCKS 3   // CTAs of 128 threads per SM the register budget targets
#endif
#ifndef K1_MIN_BLOCKS_HM
#define K1_MIN_BLOCKS_HM 3   // the same for the homogeneous-material instantiation (140 registers)
#endif
#ifndef K1_WARPS
#define K1_WARPS 4        // warps per CTA of the single-row kernel
#endif
#ifndef K1_TILE_NI
#define K1_TILE_NI 128    // columns per strip (march length)
#endif
#ifndef K1_GROUPS
#define K1_GROUPS 2       // cp.async groups of 3 columns in flight
#endif
#ifndef K1_STATIC_FIRST
#define K1_STATIC_FIRST 1     // each warp's first job = its index, its job-table entry loaded before
                              // the PDL wait; 0: every job from the queue
#endif
#ifndef K1_MARCH_UNROLL_SWE
#define K1_MARCH_UNROLL_SWE 2   // march loop unroll factor (groups of three columns) on shallow water
#endif
#ifndef K1_BULK
#define K1_BULK 0   // 1 (experiment): single-strip jobs stream their columns with TMA 1D bulk copies
                    // (cp.async.bulk + mbarrier, one elected lane) instead of per-lane cp.async
#endif
#ifndef K1_PREFETCH_CLAMP
#define K1_PREFETCH_CLAMP 1   // 1: branch-free prefetch (re-read the last column)
#endif
#ifndef K1_ALG2_AC
#define K1_ALG2_AC 3   // acoustics: bit 0 material fold, bit 1 fused update, bit 2 exponent scalings
                       // (3: measured C3 step 0.0874 vs 0.0887 ms; bit 2 adds register moves)
#endif
#ifndef K1_ALG2
#define K1_ALG2 1   // 1: fewer FP64 instructions per column on shallow water (material constants
                    // folded, fused update, limiter scalings by exponent arithmetic); measured
                    // -3% on C4, neutral-to-slower on acoustics (more register moves), so
                    // acoustics keeps the original form
#endif

namespace adj {

void fast_tile_shape(int ndim, int32_t* ni, int32_t* nj) {
    if (ndim == 2) { *ni = K1_TILE_NI; *nj = 28; } else { *ni = 256; *nj = 1; }
}

namespace fast {

constexpr unsigned FULL = 0xffffffffu;

// ADJ_STEP_COUNTER_ZERO: the last warp to leave the job queue zeroes it (and
// the exit count, and the prefill barrier) for the next launch, so no memset
// precedes a launch.
ADJ_D void release_counter(const AdjStepArgs& a, int lane, int warps) {
    if (!(a.flags & ADJ_STEP_COUNTER_ZERO) || lane != 0) return;
    if (atomicAdd(a.work_counter + 1, 1) == warps - 1) {
        a.work_counter[0] = 0;
        a.work_counter[1] = 0;
        if (a.prefill.plan.n > 0) a.work_counter[2] = 0;
    }
}

// ---- prefill: the level's planned ghost fill inside the step launch.
// Same entries and arithmetic as k2_gather (k2_ghost.cu, -fmad=false):
// unfused _rn multiplies / adds keep the values bitwise; loads bypass L1
// (ld.global.cg) so the step phase's cached loads never see a stale line.
ADJ_D double ip2(const double* p, int di, int dj, double wx, double wy) {
    const double ux = __dsub_rn(1.0, wx), uy = __dsub_rn(1.0, wy);
    double s = __dmul_rn(__dmul_rn(__ldcg(p), ux), uy);
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(__ldcg(p + di), wx), uy));
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(__ldcg(p + dj), ux), wy));
    return __dadd_rn(s, __dmul_rn(__dmul_rn(__ldcg(p + di + dj), wx), wy));
}

ADJ_D void prefill_gather(const AdjGhostPlanFillArgs& a) {
    double wt = a.w_time;
    int tmode = a.time_mode;
    if (a.w_time_dev) {           // graph replays: negative weight = old state only
        wt = __ldcg(a.w_time_dev);
        tmode = wt < 0.0 ? 0 : 1;
    }
    const int64_t cs = a.comp_stride, ccs = a.coarse_comp_stride;
    const int n = a.plan.n, nc = a.plan.nc;
    constexpr int U = 4;          // entries per thread in flight (the persistent grid is small)
    const int stride = gridDim.x * blockDim.x;
    for (int t0 = blockIdx.x * blockDim.x + threadIdx.x; t0 < n; t0 += U * stride) {
        int dst[U], src[U], cb[U], step[U];
        unsigned meta[U];
        double wx[U], wy[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + u * stride;
            const bool ok = t < n;
            const int tt = ok ? t : 0;
            dst[u] = ok ? __ldcg(a.plan.dst + tt) : -1;
            src[u] = __ldcg(a.plan.src + tt);
            meta[u] = ok ? __ldcg(a.plan.meta + tt) : 0u;
            const int ci = tt < nc ? tt : 0;
            cb[u] = nc ? __ldcg(a.plan.c_base + ci) : 0;
            step[u] = nc ? __ldcg(a.plan.c_step + ci) : 0;
            wx[u] = nc ? __ldcg(a.plan.c_wx + ci) : 0.0;
            wy[u] = nc ? __ldcg(a.plan.c_wy + ci) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + u * stride;
            if ((meta[u] & 1u) && t >= nc) {     // physical cell mirroring a coarse-interpolated ghost
                const int c0 = src[u];
                cb[u] = __ldcg(a.plan.c_base + c0); step[u] = __ldcg(a.plan.c_step + c0);
                wx[u] = __ldcg(a.plan.c_wx + c0); wy[u] = __ldcg(a.plan.c_wy + c0);
            }
        }
        double v[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (meta[u] & 1u) {
                const int di = step[u] & 0x3fffffff, dj = (int)((unsigned)step[u] >> 30);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double vo = tmode != 2 ? ip2(a.q_coarse_old + c * ccs + cb[u], di, dj, wx[u], wy[u]) : 0.0;
                    const double vn = tmode != 0 ? ip2(a.q_coarse_new + c * ccs + cb[u], di, dj, wx[u], wy[u]) : 0.0;
                    v[u][c] = tmode == 0 ? vo
                            : (tmode == 2 ? vn : __dadd_rn(__dmul_rn(__dsub_rn(1.0, wt), vo), __dmul_rn(wt, vn)));
                }
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c) v[u][c] = dst[u] >= 0 ? __ldcg(a.q + c * cs + src[u]) : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (dst[u] < 0) continue;
#pragma unroll
            for (int c = 0; c < 3; ++c)
                a.q[c * cs + dst[u]] = (meta[u] >> (1 + c)) & 1u ? __dmul_rn(v[u][c], -1.0) : v[u][c];
        }
    }
}

// ---- job fill: the level's planned ghost fill, regrouped per warp job
// (AdjJobFill).  The lanes fill the ghost cells this job's strips read, then
// the march reads them back through the shared ring.  Same entries and
// arithmetic as k2_gather; reads bypass L1 (ld.global.cg) so no line cached
// here can hold a ghost cell another warp is about to rewrite.
ADJ_D void job_fill(const AdjJobFill& f, double* q, int64_t cs, int job, int lane) {
    const int e0 = __ldg(f.entry_off + job), e1 = __ldg(f.entry_off + job + 1);
    if (e0 >= e1) return;
    double wt = f.w_time;
    int tmode = f.time_mode;
    if (f.w_time_dev) {           // graph replays: negative weight = old state only
        wt = __ldcg(f.w_time_dev);
        tmode = wt < 0.0 ? 0 : 1;
    }
    const int64_t ccs = f.coarse_comp_stride, n = f.n;
    const int mode = f.cache_mode;
    const bool coarse = f.c_base != nullptr;
    constexpr int U = 2;
    for (int t0 = e0 + lane; t0 < e1; t0 += 32 * U) {
        int dst[U], src[U], cb[U], step[U];
        unsigned meta[U];
        double wx[U], wy[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + 32 * u;
            const bool ok = t < e1;
            const int tt = ok ? t : e0;
            dst[u] = ok ? __ldg(f.dst + tt) : -1;
            src[u] = __ldg(f.src + tt);
            meta[u] = ok ? __ldg(f.meta + tt) : 0u;
            const bool lc = coarse && mode != 2;
            cb[u] = lc ? __ldg(f.c_base + tt) : 0;
            step[u] = lc ? __ldg(f.c_step + tt) : 0;
            wx[u] = lc ? __ldg(f.c_wx + tt) : 0.0;
            wy[u] = lc ? __ldg(f.c_wy + tt) : 0.0;
        }
        double v[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + 32 * u;
            if (meta[u] & 1u) {
                double vo[3], vn[3];
                if (mode == 2) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        vo[c] = tmode != 2 ? __ldcg(f.cache + c * n + t) : 0.0;
                        vn[c] = tmode != 0 ? __ldcg(f.cache + (3 + c) * n + t) : 0.0;
                    }
                } else {
                    const int di = step[u] & 0x3fffffff, dj = (int)((unsigned)step[u] >> 30);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        vo[c] = (tmode != 2 || mode == 1) ? ip2(f.q_coarse_old + c * ccs + cb[u], di, dj, wx[u], wy[u]) : 0.0;
                        vn[c] = (tmode != 0 || mode == 1) ? ip2(f.q_coarse_new + c * ccs + cb[u], di, dj, wx[u], wy[u]) : 0.0;
                    }
                    if (mode == 1) {
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            f.cache[c * n + t] = vo[c];
                            f.cache[(3 + c) * n + t] = vn[c];
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    v[u][c] = tmode == 0 ? vo[c]
                            : (tmode == 2 ? vn[c] : __dadd_rn(__dmul_rn(__dsub_rn(1.0, wt), vo[c]), __dmul_rn(wt, vn[c])));
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c) v[u][c] = dst[u] >= 0 ? __ldcg(q + c * cs + src[u]) : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (dst[u] < 0) continue;
#pragma unroll
            for (int c = 0; c < 3; ++c)
                q[c * cs + dst[u]] = (meta[u] >> (1 + c)) & 1u ? __dmul_rn(v[u][c], -1.0) : v[u][c];
        }
    }
    __threadfence_block();
}

// Software grid barrier: the persistent grid is sized to be co-resident.
ADJ_D void grid_barrier(int* counter, int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1);
        for (;;) {
            int v;
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
            if (v >= nblocks) break;
            __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

#ifndef K1_S1SUM
#define K1_S1SUM 1   // 1: wave form, s1 = (jump) - s0 (the two strengths sum to the jump of the
                     // eigen-coordinate; one FMA + one multiply fewer per face)
#endif
#ifndef K1_SHFL_K1
#define K1_SHFL_K1 0   // 1: the upper cell's 1 + m^2 by shuffle instead of recomputed
#endif
#ifndef K1_RCP_CUBIC
#define K1_RCP_CUBIC 1   // 0: one quadratic Newton step (relative error ~e^2)
#endif
#ifndef K1_PRED_STORE
#define K1_PRED_STORE 0   // 1: the update runs on every lane, only its stores are predicated by out_lane
#endif
ADJ_D void st_pred(double* p, double v, bool pred) {   // st.global.f64 under a predicate (no branch)
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}\n" ::"l"(p), "d"(v),
                 "r"((int)pred) : "memory");
}

ADJ_D double rcp(double x) {  // x > 0, normal: MUFU seed + one cubic Newton step
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
#if K1_RCP_CUBIC
    return fma(r, fma(e, e, e), r);   // r (1 + e + e^2): relative error ~e^3
#else
    return fma(r, e, r);
#endif
}

ADJ_D double dmin(double a, double b) { return a < b ? a : b; }
ADJ_D double dmax(double a, double b) { return a > b ? a : b; }

// 2^k v for a finite v by adding k to the exponent field (integer pipe; the sign bit is untouched).
// Exact for normal results; v == 0 gives 2^(k-1023) (~1e-308), which the
// limiters below only ever compare against or scale by O(1) coefficients.
template <int K, bool ALG>
ADJ_D double pow2x(double v) {
    if (ALG) return __hiloint2double(__double2hiint(v) + (K << 20), __double2loint(v));
    return (double)(1 << K) * v;
}

ADJ_D double sh_dn(double v) { return __shfl_down_sync(FULL, v, 1); }  // from lane+1 (row j+1)
ADJ_D double sh_up(double v) { return __shfl_up_sync(FULL, v, 1); }    // from lane-1 (row j-1)

// Division-free limited strength, doubled: 2 phi(B/A) A (solver.py:65-77).
// With theta = B/A, phi(theta) A is 0 when A, B have opposite signs and
// otherwise sign(A) times  MC: min(|A+B|/2, 2|A|, 2|B|);  minmod: min(|A|,|B|);
// superbee: max(min(|A|, 2|B|), min(2|A|, |B|)).  The factor 1/2 is folded
// into the per-cell 1/(2(1+m^2)) the result is multiplied by.
//
// Evaluated in the signed domain: when A and B share a sign, every candidate
// (A, B, A+B and their power-of-two multiples) carries that sign, so the
// selections compare magnitudes through DSETP's |.| operand modifiers and pick
// the signed value -- no |x| is materialised (each one was an FP64 DADD) and
// no copysign is needed.  Same selections as the magnitude form, so the same
// values bit for bit.
template <int LIM, bool ALG>
ADJ_D double limab2(double A, double B) {
    double r;
    if (LIM == ADJ_LIM_MINMOD) {
        const double m = fabs(A) < fabs(B) ? A : B;
        r = m + m;
    } else if (LIM == ADJ_LIM_MC) {
        const double m4 = pow2x<2, ALG>(fabs(A) < fabs(B) ? A : B);
        const double S = __dadd_rn(A, B);   // A, B are products: no contraction (see correction())
        r = fabs(S) < fabs(m4) ? S : m4;
    } else {
        const double A2 = pow2x<1, ALG>(A), B2 = pow2x<1, ALG>(B);
        const double A4 = pow2x<2, ALG>(A), B4 = pow2x<2, ALG>(B);
        const double t1 = fabs(A2) < fabs(B4) ? A2 : B4;
        const double t2 = fabs(A4) < fabs(B2) ? A4 : B2;
        r = fabs(t1) > fabs(t2) ? t1 : t2;
    }
    return (__double2hiint(A) ^ __double2hiint(B)) < 0 ? 0.0 : r;
}

// Per-cell material quantities.  m: eigen material (z for acoustics, c for
// shallow water); k1i = 1/(2(1+m^2)); kx, ky: correction magnitudes
// (wave: 0.5 c (1 - dtd c); f-wave: 0.5 (1 - dtd c)); tr: transverse helper
// (acoustics K = c z, shallow water c^2); fx: f-wave flux factor (acoustics
// 1/rho, shallow water g h = c^2).
struct Mat {
    double c, m, k1, k1i, kx, ky, tr, fx;   // k1 = 1+m^2, k1i = 1/(2 k1); kx, ky include k1i when limited
};

template <int SYS, int FORM, int LIM, bool SQ = false>
ADJ_D Mat make_mat(double c, double z, double dtdx, double dtdy) {   // SQ: dtdx == dtdy, so ky == kx
    constexpr bool SWE = SYS == ADJ_SYS_SWE2D, FW = FORM == ADJ_FORM_FWAVE;
    Mat t;
    t.c = c;
    t.m = SWE ? c : z;
    t.k1 = fma(t.m, t.m, 1.0);
    if (K1_ALG2 && (SWE || (K1_ALG2_AC & 1))) {
    // the limited strength is only ever used scaled by k / (2 (1 + m^2)), with
    // k = (c) 0.5 (1 - dtd c): fold both halves into 0.25 (1 - dtd c) / (1 + m^2)
    if (LIM != ADJ_LIM_NONE) {
        const double r = rcp(t.k1);
        const double ck = FW ? r : c * r;
        t.k1i = 0.5 * r;
        t.kx = ck * fma(-0.25 * dtdx, c, 0.25);
        t.ky = SQ ? t.kx : ck * fma(-0.25 * dtdy, c, 0.25);
    } else {
        t.kx = FW ? fma(-0.5 * dtdx, c, 0.5) : c * fma(-0.5 * dtdx, c, 0.5);
        t.ky = SQ ? t.kx : (FW ? fma(-0.5 * dtdy, c, 0.5) : c * fma(-0.5 * dtdy, c, 0.5));
    }
    } else {
    const double hx = 0.5 * fma(-dtdx, c, 1.0), hy = SQ ? hx : 0.5 * fma(-dtdy, c, 1.0);
    t.kx = FW ? hx : c * hx;
    t.ky = SQ ? t.kx : (FW ? hy : c * hy);
    if (LIM != ADJ_LIM_NONE) {   // the limited strength is only ever used scaled by k / (2 (1 + m^2))
        t.k1i = rcp(t.k1 + t.k1);
        t.kx *= t.k1i;
        t.ky = SQ ? t.kx : t.ky * t.k1i;
    }
    }
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
            f.s1 = K1_S1SUM ? dn - f.s0 : (L.m * dn + d0) * inv;
            // amdq = -cL W1 = s0 (cL zL, -cL) ; apdq = cR W2 = s1 (cR zR, cR)
            f.am0 = f.s0 * L.tr; f.am1 = -f.s0 * L.c;
            f.ap0 = f.s1 * R.tr; f.ap1 = f.s1 * R.c;
        } else {          // swe_linear_rp
            f.s0 = (R.c * d0 - dn) * inv;
            f.s1 = K1_S1SUM ? d0 - f.s0 : (L.c * d0 + dn) * inv;
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

// Shallow water with dry cells (_swe_effective_states, solver.py:357-380): a
// dry side takes the wet side's state with the normal momentum negated and the
// wet side's material; a both-dry face has no waves (zero strengths and
// fluctuations).  wet <=> c > 0 (SweMaterial.create: c = sqrt(g max(depth, 0))).
// The solve itself is the regular one on the effective states and materials
// (forward wave form and the time-reversed f-wave adjoint).
template <int SYS, int FORM, bool REV>
ADJ_D Face solve_face_wd(double qL0, double qLn, double qR0, double qRn, double cL, double cR, bool wl, bool wr) {
    const double a0 = wl ? qL0 : qR0, an = wl ? qLn : -qRn;
    const double b0 = wr ? qR0 : qL0, bn = wr ? qRn : -qLn;
    const bool dd = !wl && !wr;
    const double cl = wl ? cL : (wr ? cR : 1.0), cr = wr ? cR : (wl ? cL : 1.0);   // dd: finite dummies
    Mat Le{}, Re{};
    Le.c = Le.m = cl;
    Re.c = Re.m = cr;
    Le.tr = Le.fx = cl * cl;   // shallow water: c^2 = g h (transverse helper and f-wave flux factor)
    Re.tr = Re.fx = cr * cr;
    Face f = solve_face<SYS, FORM, REV>(a0, an, b0, bn, Le, Re);
    if (dd) { f.s0 = f.s1 = 0.0; f.am0 = f.am1 = f.ap0 = f.ap1 = 0.0; }
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
    // Products that feed both a sum and another use are written with explicit roundings, so that
    // which of them fuses into the sum (FMA contraction) is not the compiler's choice per
    // instantiation.  (Other contractions still differ between instantiations -- e.g. the
    // transverse products the homogeneous march shares -- so instantiations agree to rounding,
    // not bitwise.)
    if (LIM == ADJ_LIM_NONE) {
        p0 = f.s0; p1 = f.s1;
    } else {
        const double A0 = __dmul_rn(f.s0, L.k1);
        const double A1 = __dmul_rn(f.s1, R.k1);
        const double B0 = __dmul_rn(s0_nb, REV ? P0_nb : f.P);
        const double B1 = __dmul_rn(s1_nb, REV ? P1_nb : f.P);
        p0 = limab2<LIM, K1_ALG2 && (SWE || (K1_ALG2_AC & 4))>(A0, B0);   // 1/(2(1+m^2)) folded into kL, kR
        p1 = limab2<LIM, K1_ALG2 && (SWE || (K1_ALG2_AC & 4))>(A1, B1);
    }
    // coefficients: wave 0.5|s|(1-dtd|s|) for both; f-wave sign(s) 0.5(1-dtd|s|)
    const double u0 = __dmul_rn(FW ? -kL : kL, p0);
    const double u1 = __dmul_rn(kR, p1);
    const double mL = SWE ? L.c : L.m, mR = SWE ? R.c : R.m;
    const double dif = fma(mR, u1, -__dmul_rn(mL, u0)), sum = __dadd_rn(u0, u1);
    if (MPOS0) { F0 = dif; Fn = sum; }
    else { F0 = sum; Fn = dif; }
}

// Transverse split of an entering fluctuation (component 0 = f0; its
// transverse component is zero for every 2D system here), scaled by h.
// Returns bm (to the lower transverse face) and bp (upper), components
// (0, transverse velocity) -- bm's component 0 NEGATED (nbm0 = -bm0): for
// shallow water it is the product u itself, and the callers subtract it
// (x - y == x + (-y) exactly), so no negation is materialised before the
// shuffle that carries it.
template <int SYS, int FORM, bool REV>
ADJ_D void transverse(double f0, double h, const Mat& b, const Mat& a,
                      double& nbm0, double& bmv, double& bp0, double& bpv) {
    constexpr bool SWE = SYS == ADJ_SYS_SWE2D, FW = FORM == ADJ_FORM_FWAVE;
    const double t = (h * f0) * rcp(b.m + a.m);
    double nm0, mv, p0, pv;   // nm0 = -m0
    if (!FW) {
        if (!SWE) { nm0 = b.tr * t; mv = b.c * t; p0 = a.tr * t; pv = a.c * t; }
        else { const double u = (b.c * a.c) * t; nm0 = u; mv = b.c * u; p0 = u; pv = a.c * u; }
    } else {
        if (!SWE) { const double ta = a.m * t, tb = b.m * t; nm0 = b.c * ta; mv = b.tr * ta; p0 = a.c * tb; pv = a.tr * tb; }
        else { nm0 = b.tr * t; mv = b.c * t; p0 = a.tr * t; pv = a.c * t; }
    }
    if (REV) { nbm0 = p0; bmv = -pv; bp0 = nm0; bpv = -mv; }
    else { nbm0 = nm0; bmv = mv; bp0 = p0; bpv = pv; }
}

struct Raw { double q0, q1, q2, c, z; };

#ifndef K1_LDSNB
#define K1_LDSNB 0   // 1: y-neighbours' raw q and material read from the shared ring (LDS.64)
                     // instead of warp shuffles; the ring keeps the current and previous
                     // column groups resident, so it has GROUPS + 2 groups
#endif
constexpr int GROUPS = K1_GROUPS;  // cp.async groups (of 3 columns) in flight per warp
constexpr int RING = 3 * GROUPS;   // column slots of the two-row kernel's ring
constexpr int NGRP = K1_LDSNB ? GROUPS + 2 : GROUPS;   // groups of the single-row kernel's ring
constexpr int RING1 = 3 * NGRP;

// One warp's march along x over an output strip.  Every carried quantity
// lives in a 3-slot ring indexed by (column mod 3); column<K> is the body of
// the march for a column in slot K, so the 3-way unrolled loop rotates roles
// by renaming instead of moving registers.
// HM: homogeneous material (ADJ_STEP_UNIFORM_MAT) -- every cell of the level has the material
// (uniform_c, uniform_z), so the per-cell material quantities, the face and transverse
// reciprocals and 1 + mL mR are loop invariants of the march (computed once per strip by the same
// functions on the same values: bitwise equal to the per-cell form), no material plane is
// loaded and no material crosses lanes.
template <int SYS, int FORM, bool REV, int LIM, bool CFL, bool RST = false, bool SQ = false, bool WD = false,
          bool HM = false>
struct Strip {
    static constexpr bool SWE = SYS == ADJ_SYS_SWE2D;
    static constexpr bool FWD_WAVE = FORM == ADJ_FORM_WAVE && !REV;
    static constexpr int MARCH_UNROLL = SWE && !WD ? K1_MARCH_UNROLL_SWE : 1;
    const double* __restrict__ qin;
    const double* __restrict__ aux;
    double* __restrict__ qout;
    int64_t cs, as;
    int pitch, g, i0, ni, s_last, colbase;   // s: column relative to the strip (i0 = 0)
    bool out_lane, yface_cfl;
    double dtdx, dtdy, hx, hy;

    double* ring;                  // this warp's cp.async ring: [RING1][NARR][32]
#if K1_BULK
    bool bulk;                     // this job streams by bulk copies (a single strip on lanes 0..31)
    unsigned mbar;                 // shared address of this warp's GROUPS mbarriers
    unsigned* phase;               // per-warp parity bits of the mbarriers (persist across jobs)
    const double* seg;             // lane 0's row of q_in / aux (segment start), unclamped rows follow
    const double* segaux;

    // three columns s0.. into slots slot0.. (group g): one expect_tx, 3 * NARR copies of 256 bytes
    ADJ_D void prefetch_group(int s0, int slot0, int g) const {
        if (lane == 0) {
            const unsigned bar = mbar + 8u * g;
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(3 * NARR * 256)
                         : "memory");
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int sc = s0 + k < s_last ? s0 + k : s_last;
                const int64_t o = (int64_t)(colbase + sc) * pitch;
                const double* src[5] = {seg + o, seg + cs + o, seg + 2 * cs + o, segaux + o, segaux + as + o};
#pragma unroll
                for (int a_ = 0; a_ < NARR; ++a_) {
                    const unsigned dst = (unsigned)__cvta_generic_to_shared(ring + ((slot0 + k) * NARR + a_) * 32);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];\n" ::"r"(dst),
                        "l"(src[a_]), "r"(bar)
                        : "memory");
                }
            }
        }
    }
    ADJ_D void wait_group_bulk(int g) const {
        const unsigned bar = mbar + 8u * g, par = (*phase >> g) & 1u;
        unsigned done = 0;
        for (int spin = 0; !done; ++spin) {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(bar), "r"(par) : "memory");
            if (spin > (1 << 24)) __trap();      // experiment guard: never hang the device
        }
        *phase ^= 1u << g;
    }
#endif
    int lane, lup, ldn;            // lane, and the lanes of rows j+1, j-1 (clamped like the shuffles)
    Mat m[3];
    Mat mh;                        // HM: the level's material
    double q0[3], q1[3], q2[3];
    Face xf[3];                    // xf[k]: x-face left of column k
    double sy0[3], sy2[3];         // Sy(column)
    double gt0[3], gt2[3];         // gtil, own top face, of column
    double cy0[3], cy2[3];         // limited y correction of column
    double bpy0[3], bpy1[3];       // bp of transverse(Sy(column))
    double ft0[3], ft1[3];         // ftil at the x-face left of column
    double sx0[3], sx1[3];         // Sx(column)
    double cup[3], mup[3];         // row j+1 materials of column (WD: transverse materials)
    // WD (shallow water with dry cells, forward wave form): per-column wet
    // flags of this row, wet-wet flag of the y-face above, transverse
    // material (dry cells at unit depth: sqrt(g), _swe_transverse_material)
    bool wet[3], wwy[3];
    double tcv[3], sqrtg;
    double smx, smy;
    unsigned bad;
    // fused restriction (RST): block sums of the new values over R rows x R columns
    double ra0, ra1, ra2;
    double* rq;                    // coarse state
    const int32_t* rcell;
    int64_t rcs;
    int rr, rx0, rbase, rnyb, rby;  // ratio, strip x origin, patch block base, blocks per row, block row
    bool rlead;                     // first row of an output block

    static constexpr int NARR = HM ? 3 : (SWE ? 4 : 5);

    // issue the cp.async copies of column s into ring slot `slot`
    ADJ_D void prefetch(int s, int slot) const {
#if K1_PREFETCH_CLAMP   // branch-free: columns past the strip re-read its last column, unused
        {
            const int sc = s < s_last ? s : s_last;
#else
        if (s <= s_last) {
            const int sc = s;
#endif
            const int64_t o = (int64_t)(colbase + sc) * pitch;
            const double* src[5] = {qin + o, qin + cs + o, qin + 2 * cs + o, aux + o, aux + as + o};
#pragma unroll
            for (int k = 0; k < NARR; ++k) {
                const unsigned dst = (unsigned)__cvta_generic_to_shared(ring + (slot * NARR + k) * 32 + lane);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src[k]) : "memory");
            }
        }
    }

    ADJ_D static void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

    ADJ_D Raw read(int slot) const {
        const double* r = ring + slot * NARR * 32 + lane;
        Raw v;
        v.q0 = r[0]; v.q1 = r[32]; v.q2 = r[64];
        if (HM) { v.c = mh.c; v.z = mh.m; }
        else { v.c = r[96]; v.z = SWE ? 0.0 : r[128]; }
        return v;
    }

    // up: this column's ring slot at the lane of row j+1; dn: the previous
    // column's slot at the lane of row j-1 (array k at +32k)
    template <int K>
    ADJ_D void column(int s, const Raw& cr, const double* up, const double* dn) {
        constexpr int C = K, P = (K + 2) % 3, PP = (K + 1) % 3;
        if (!HM) m[C] = make_mat<SYS, FORM, LIM, SQ>(cr.c, cr.z, dtdx, dtdy);   // HM: m[] = mh throughout
        if (WD) {
            wet[C] = __double2hiint(cr.c) > 0;   // c >= 0: c > 0 <=> its high word is positive
            tcv[C] = wet[C] ? cr.c : sqrtg;
        }
        // CFL: max |speed| of the faces is the max material speed of the cells
        // they touch (fast path = no dry cells): x-faces of this strip touch
        // columns [i0-1, i0+ni] of the output rows, y-faces rows j0-1..j0+nj
        // of the output columns (solver.py:457-460)
        if (CFL) {
            if (s >= i0 - 1 && s <= i0 + ni && out_lane) smx = cr.c > smx ? cr.c : smx;
            if (s >= i0 && s < i0 + ni && yface_cfl) smy = cr.c > smy ? cr.c : smy;
        }
        q0[C] = cr.q0; q1[C] = cr.q1; q2[C] = cr.q2;

        // ---- x-face s-1/2 between columns s-1 and s
        if (WD) xf[C] = solve_face_wd<SYS, FORM, REV>(q0[P], q1[P], cr.q0, cr.q1, m[P].c, m[C].c, wet[P], wet[C]);
        else xf[C] = solve_face<SYS, FORM, REV>(q0[P], q1[P], cr.q0, cr.q1, m[P], m[C]);

        // ---- y-face between rows j and j+1 at column s
        const double uq0 = K1_LDSNB ? up[0] : sh_dn(cr.q0);
        const double uq2 = K1_LDSNB ? up[64] : sh_dn(cr.q2);
        Mat mu{};
        if (HM) {
            mu = mh;
        } else {
            mu.c = K1_LDSNB ? up[96] : sh_dn(m[C].c);
            mu.m = SWE ? mu.c : (K1_LDSNB ? up[128] : sh_dn(m[C].m));
            mu.k1 = K1_SHFL_K1 ? sh_dn(m[C].k1) : fma(mu.m, mu.m, 1.0);
            mu.ky = sh_dn(m[C].ky);
            mu.kx = 0.0;
            mu.tr = SWE ? mu.c * mu.c : mu.c * mu.m;
            mu.fx = FORM == ADJ_FORM_FWAVE ? sh_dn(m[C].fx) : 0.0;
        }
        const bool wu = WD ? __double2hiint(mu.c) > 0 : true;
        const Face yf = WD ? solve_face_wd<SYS, FORM, REV>(cr.q0, cr.q2, uq0, uq2, m[C].c, mu.c, wet[C], wu)
                           : solve_face<SYS, FORM, REV>(cr.q0, cr.q2, uq0, uq2, m[C], mu);
        if (WD) wwy[C] = wet[C] && wu;
        const double s1up = REV ? 0.0 : sh_up(yf.s1);   // forward: the family-1 limiter neighbour and Sy's s1 below
        {
            const double s0n = REV ? sh_up(yf.s0) : sh_dn(yf.s0);
            const double s1n = REV ? sh_dn(yf.s1) : s1up;
            const double P0n = REV ? sh_up(yf.P) : 0.0;
            const double P1n = REV ? sh_dn(yf.P) : 0.0;
            correction<SYS, FORM, REV, LIM>(yf, s0n, P0n, s1n, P1n, m[C], mu, m[C].ky, mu.ky, cy0[C], cy2[C]);
        }
        if (FWD_WAVE) {
            // Sy(cell) = apdq(face below, R = cell) + amdq(own face, L = cell): the
            // cell's own material times the two strengths (s1 below is the
            // limiter neighbour the correction above already shuffled)
            const double s1b = s1up;
            if (SWE) { sy0[C] = m[C].c * (s1b - yf.s0); sy2[C] = m[C].tr * (s1b + yf.s0); }
            else { sy0[C] = m[C].tr * (s1b + yf.s0); sy2[C] = m[C].c * (s1b - yf.s0); }
        } else {
            sy0[C] = yf.am0 + sh_up(yf.ap0);
            sy2[C] = yf.am1 + sh_up(yf.ap1);
        }
        cup[C] = WD ? sh_dn(tcv[C]) : mu.c;
        mup[C] = WD ? cup[C] : mu.m;

        // ---- Sx(s-1) and its transverse split with rows j-1, j+1 of column s-1
        if (FWD_WAVE) {   // Sx(s-1) from the strengths of its two x-faces and its own material
            const double sl = xf[P].s1, sr = xf[C].s0;
            if (SWE) { sx0[P] = m[P].c * (sl - sr); sx1[P] = m[P].tr * (sl + sr); }
            else { sx0[P] = m[P].tr * (sl + sr); sx1[P] = m[P].c * (sl - sr); }
        } else {
            sx0[P] = xf[P].ap0 + xf[C].am0;
            sx1[P] = xf[P].ap1 + xf[C].am1;
        }
        {
            Mat mb{}, ma{};
            if (HM) {
                mb = mh; ma = mh;
            } else {
                mb.c = WD ? sh_up(tcv[P]) : (K1_LDSNB ? dn[96] : sh_up(m[P].c));
                mb.m = SWE ? mb.c : (K1_LDSNB ? dn[128] : sh_up(m[P].m));
                mb.tr = SWE ? mb.c * mb.c : mb.c * mb.m;
                ma.c = cup[P]; ma.m = mup[P];
                ma.tr = SWE ? ma.c * ma.c : ma.c * ma.m;
            }
            double nbm0, bmv, bp0, bpv;
            transverse<SYS, FORM, REV>(sx0[P], hx, mb, ma, nbm0, bmv, bp0, bpv);
            gt0[P] = cy0[P] - (bp0 - sh_dn(nbm0));
            gt2[P] = cy2[P] - (bpv + sh_dn(bmv));
            if (WD && !wwy[P]) gt0[P] = gt2[P] = 0.0;   // gtil[:, ~wwy] = 0 (solver.py:500-502)
        }

        // ---- transverse of Sy(s-1) with columns s-2, s; x-limiter of face s-3/2
        {
            double nbm0, bmv, bp0, bpv;
            if (WD) {
                Mat tb{}, ta{};
                tb.c = tb.m = tcv[PP];
                ta.c = ta.m = tcv[C];
                tb.tr = tb.c * tb.c;   // shallow water: c^2 (the f-wave transverse uses it)
                ta.tr = ta.c * ta.c;
                transverse<SYS, FORM, REV>(sy0[P], hy, tb, ta, nbm0, bmv, bp0, bpv);
            } else {
                transverse<SYS, FORM, REV>(sy0[P], hy, m[PP], m[C], nbm0, bmv, bp0, bpv);
            }
            double fc0, fc1;
            correction<SYS, FORM, REV, LIM>(xf[P], REV ? xf[PP].s0 : xf[C].s0, xf[PP].P,
                                            REV ? xf[C].s1 : xf[PP].s1, xf[C].P,
                                            m[PP], m[P], m[PP].kx, m[P].kx, fc0, fc1);
            ft0[P] = fc0 - (bpy0[PP] - nbm0);
            ft1[P] = fc1 - (bpy1[PP] + bmv);
            if (WD && !(wet[PP] && wet[P])) ft0[P] = ft1[P] = 0.0;   // ftil[:, ~wwx] = 0
            bpy0[P] = bp0; bpy1[P] = bpv;
        }

        // ---- update cell s-2
        const double gb0 = sh_up(gt0[PP]), gb2 = sh_up(gt2[PP]);
#if K1_PRED_STORE
        if (s >= i0 + 2 && s <= s_last) {   // warp-uniform; only the stores are per lane (predicated)
#else
        if (s >= i0 + 2 && s <= s_last && out_lane) {
#endif
            double n0, n1, n2;
            if (K1_ALG2 && (SWE || (K1_ALG2_AC & 2))) {
                n0 = fma(-dtdy, (sy0[PP] + gt0[PP]) - gb0, fma(-dtdx, (sx0[PP] + ft0[P]) - ft0[PP], q0[PP]));
                n1 = fma(-dtdx, (sx1[PP] + ft1[P]) - ft1[PP], q1[PP]);
                n2 = fma(-dtdy, (sy2[PP] + gt2[PP]) - gb2, q2[PP]);
            } else {
                const double d0 = -dtdx * ((sx0[PP] + ft0[P]) - ft0[PP]) - dtdy * ((sy0[PP] + gt0[PP]) - gb0);
                const double d1 = -dtdx * ((sx1[PP] + ft1[P]) - ft1[PP]);
                const double d2 = -dtdy * ((sy2[PP] + gt2[PP]) - gb2);
                n0 = q0[PP] + d0; n1 = q1[PP] + d1; n2 = q2[PP] + d2;
            }
            if (WD && !wet[PP]) { n0 = q0[PP]; n1 = q1[PP]; n2 = q2[PP]; }   // dq *= wet
            const int64_t o = (int64_t)(colbase + s - 2) * pitch;
            // non-finite <=> exponent bits all set (integer pipe)
            const unsigned ex = 0x7ff00000u;
            const bool nf = (((unsigned)__double2hiint(n0) & ex) == ex) | (((unsigned)__double2hiint(n1) & ex) == ex) |
                            (((unsigned)__double2hiint(n2) & ex) == ex);
#if K1_PRED_STORE
            st_pred(qout + o, n0, out_lane); st_pred(qout + cs + o, n1, out_lane); st_pred(qout + 2 * cs + o, n2, out_lane);
            bad |= out_lane & nf;
            if (RST) { ra0 += out_lane ? n0 : 0.0; ra1 += out_lane ? n1 : 0.0; ra2 += out_lane ? n2 : 0.0; }
#else
            qout[o] = n0; qout[cs + o] = n1; qout[2 * cs + o] = n2;
            bad |= nf;
            if (RST) { ra0 += n0; ra1 += n1; ra2 += n2; }
#endif
        }
        if (RST && s >= i0 + 2 && s <= s_last && ((s - 2) & (rr - 1)) == rr - 1) {   // warp-uniform
            // sum the block's R rows (lanes), then its leader lane writes the mean
            double v0 = ra0 + sh_dn(ra0), v1 = ra1 + sh_dn(ra1), v2 = ra2 + sh_dn(ra2);
            if (rr == 4) {
                v0 += __shfl_down_sync(FULL, v0, 2);
                v1 += __shfl_down_sync(FULL, v1, 2);
                v2 += __shfl_down_sync(FULL, v2, 2);
            }
            if (rlead) {
                const int dst = __ldg(rcell + rbase + ((rx0 + s - 2) / rr) * rnyb + rby);
                if (dst >= 0) {
                    const double inv = rr == 4 ? 0.0625 : 0.25;   // np.mean: sum / r^2 (a power of two)
                    rq[dst] = v0 * inv; rq[rcs + dst] = v1 * inv; rq[2 * rcs + dst] = v2 * inv;
                }
            }
            ra0 = ra1 = ra2 = 0.0;
        }
    }

    // Lane setup for a strip T placed at lanes [lane0, lane0 + nj + 4).
    ADJ_D void setup(const AdjTile& T, const AdjPatch& p, const AdjStepArgs& a, int lane_, int lane0,
                     double* ring_, double hc = 0.0, double hz = 0.0) {
        lane = lane_;
        lup = lane < 31 ? lane + 1 : 31;
        ldn = lane > 0 ? lane - 1 : 0;
        ring = ring_;
        g = a.ghost;
        const int l = lane - lane0;
        const int NY = p.ny + 2 * g;
        const int jj = g + T.j0 - 2 + l;
        const int jl = jj < 0 ? 0 : (jj > NY - 1 ? NY - 1 : jj);
        out_lane = l >= 2 && l < 2 + T.nj;
        yface_cfl = l >= 1 && l < 3 + T.nj;
        cs = a.comp_stride; as = a.aux_stride;
        qin = a.q_in + p.offset + jl;
        aux = a.aux + p.offset + jl;
        qout = a.q_out + p.offset + jl;
        pitch = p.pitch;
        dtdx = a.dtdx; dtdy = a.dtdy;
        hx = 0.5 * dtdx; hy = 0.5 * dtdy;
        sqrtg = WD ? sqrt(a.gravity) : 0.0;
        if (HM) mh = make_mat<SYS, FORM, LIM, SQ>(hc, hz, dtdx, dtdy);
        colbase = g + T.i0;
        i0 = 0; ni = T.ni;
#if K1_BULK
        seg = a.q_in + p.offset + (g + T.j0 - 2);
        segaux = a.aux + p.offset + (g + T.j0 - 2);
#endif
        if (RST) {
            const AdjStepRestrict& R = a.fine_restrict;
            ra0 = ra1 = ra2 = 0.0;
            rq = R.q_coarse; rcell = R.cell; rcs = R.coarse_comp_stride; rr = R.ratio;
            rx0 = T.i0;
            rbase = __ldg(R.base + T.patch);
            rnyb = p.ny / rr;
            const int jr = T.j0 + l - 2;           // interior row of this lane
            rby = jr >= 0 ? jr / rr : 0;
            rlead = out_lane && jr % rr == 0;
        }
    }

    template <int UNR = MARCH_UNROLL>
    ADJ_D void run() {
        const int s_first = -2;
        s_last = ni + 1;
#if K1_BULK
        const bool bk = bulk;
#else
        constexpr bool bk = false;
#endif
#pragma unroll
        for (int gI = 0; gI < GROUPS; ++gI) {
#if K1_BULK
            if (bk) { prefetch_group(s_first + 3 * gI, 3 * gI, gI); continue; }
#endif
            for (int k = 0; k < 3; ++k) prefetch(s_first + 3 * gI + k, 3 * gI + k);
            commit();
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            m[k] = HM ? mh : Mat{}; xf[k] = Face{};
            q0[k] = q1[k] = q2[k] = 0.0;
            sy0[k] = sy2[k] = gt0[k] = gt2[k] = cy0[k] = cy2[k] = 0.0;
            bpy0[k] = bpy1[k] = ft0[k] = ft1[k] = sx0[k] = sx1[k] = cup[k] = mup[k] = 0.0;
            if (WD) { wet[k] = wwy[k] = false; tcv[k] = 0.0; }
        }
        // columns beyond s_last (at most two, rounding the march to whole
        // rotations) compute on stale registers and write nothing
        int base = 0;
        // shallow water: six columns per loop body (fewer loop-carried register moves, 253 -> 244
        // instructions per column; C4 K1 0.2127 -> 0.2110 ms); acoustics measured neutral-to-slower
#pragma unroll(UNR)
        for (int s = s_first; s <= s_last; s += 3) {
            // one wait per group of three columns, then the columns 3*GROUPS
            // ahead go to the group after the in-flight ones (with K1_LDSNB the
            // current and previous groups stay resident for neighbour reads)
#if K1_BULK
            if (bk) wait_group_bulk(base / 3);
            else
#endif
            asm volatile("cp.async.wait_group %0;\n" ::"n"(GROUPS - 1) : "memory");
            const Raw r0 = read(base), r1 = read(base + 1), r2 = read(base + 2);
            int pf = base + 3 * GROUPS;
            if (pf >= RING1) pf -= RING1;
#if K1_BULK
            if (bk) {
                __syncwarp();                      // every lane has read the group before it is overwritten
                prefetch_group(s + 3 * GROUPS, pf, pf / 3);
            } else
#endif
            {
            prefetch(s + 3 * GROUPS, pf);
            prefetch(s + 3 * GROUPS + 1, pf + 1);
            prefetch(s + 3 * GROUPS + 2, pf + 2);
            commit();
            }
            constexpr int SL = NARR * 32;          // doubles per column slot
            const double* rb = ring + base * SL;
            const double* rp = (base == 0 ? ring + RING1 * SL : rb) - SL;   // slot before base
            column<0>(s, r0, rb + lup, rp + ldn);
            column<1>(s + 1, r1, rb + SL + lup, rb + ldn);
            column<2>(s + 2, r2, rb + 2 * SL + lup, rb + SL + ldn);
            base = base + 3 == RING1 ? 0 : base + 3;
        }
#if K1_BULK
        if (bk) {   // the groups prefetched past the strip's end
            for (int gI = 0; gI < GROUPS; ++gI) {
                wait_group_bulk(base / 3);
                base = base + 3 == RING1 ? 0 : base + 3;
            }
            __syncwarp();
            return;
        }
#endif
        asm volatile("cp.async.wait_all;\n" ::: "memory");
    }
};

// A strip whose output cells are all dry: dq *= wet leaves them unchanged, so
// the step copies them (every lane its row, column by column, coalesced).
// Returns whether a copied value is non-finite (the reference's q + 0 dq).
ADJ_D bool dry_copy(const AdjStepArgs& a, const AdjTile& T, const AdjPatch& p, int lane, int lane0) {
    const int l = lane - lane0;
    if (l < 2 || l >= 2 + T.nj) return false;
    const int g = a.ghost;
    const int64_t cs = a.comp_stride;
    const int64_t base = p.offset + (int64_t)(g + T.i0) * p.pitch + (g + T.j0 + l - 2);
    bool bad = false;
    for (int i = 0; i < T.ni; ++i) {
        const int64_t o = base + (int64_t)i * p.pitch;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double v = __ldg(a.q_in + c * cs + o);
            a.q_out[c * cs + o] = v;
            bad |= (((unsigned)__double2hiint(v) & 0x7ff00000u) == 0x7ff00000u);
        }
    }
    return bad;
}

// ---- ADJ_STEP_PHYS_IN: fill_ghost_physical of q_in inside the step launch.
// One patch spanning the level, ghost width 2.  A ghost-inclusive index ii
// on an axis of n interior cells maps to its interior source and a wall sign
// (solver.py:84-122; periodic wraps); a corner takes the x rule then the y
// rule, as the x-slab-then-y-slab fill leaves it.
ADJ_D int phys_src(int ii, int n, int bclo, int bchi, bool& neg) {
    const int i = ii - 2;
    if (i < 0) {
        const int k = -i;
        neg = bclo == ADJ_BC_WALL;
        return bclo == ADJ_BC_OUTFLOW ? 0 : (bclo == ADJ_BC_WALL ? k - 1 : n - k);
    }
    if (i >= n) {
        const int k = i - n + 1;
        neg = bchi == ADJ_BC_WALL;
        return bchi == ADJ_BC_OUTFLOW ? n - 1 : (bchi == ADJ_BC_WALL ? n - k : k - 1);
    }
    neg = false;
    return i;
}

// The ghost cells of strip T's read window (ghost-inclusive rows T.j0 ..
// T.j0 + nj + 3, columns T.i0 .. T.i0 + ni + 3), spread over the warp's lanes.
// Sources are interior cells (not written by this launch); a ghost cell in two
// windows gets the same value from both jobs.  Strips away from the domain
// sides have no ghost cells in their window and return at once.
ADJ_D void phys_prefill(const AdjStepArgs& a, const AdjTile& T, const AdjPatch& p, int lane) {
    const int nx = p.nx, ny = p.ny;
    const int r0 = T.j0, r1 = min(T.j0 + T.nj + 4, ny + 4);
    const int c0 = T.i0, c1 = min(T.i0 + T.ni + 4, nx + 4);
    const int glo = max(0, min(2, r1) - r0), ghi = max(0, r1 - max(r0, ny + 2));
    const int clo = max(0, min(2, c1) - c0), chi = max(0, c1 - max(c0, nx + 2));
    const int gr = glo + ghi, gc = clo + chi, Wc = c1 - c0, Wr = r1 - r0;
    const int G = gr * Wc + gc * (Wr - gr);
    if (G == 0) return;
    double* q = const_cast<double*>(a.q_in) + p.offset;
    const int64_t cs = a.comp_stride;
    const int nnx = a.phys_normal[0], nny = a.phys_normal[1];
    constexpr int U = 4;                           // cells per lane with their loads in flight together
    for (int e0 = lane; e0 < G; e0 += 32 * U) {
        int64_t dst[U];
        unsigned neg[U];
        double v[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + 32 * u;
            int ii, jj;
            if (e < gr * Wc) {                     // ghost rows (y sides), every window column
                const int rr = e / Wc;
                jj = rr < glo ? r0 + rr : max(r0, ny + 2) + (rr - glo);
                ii = c0 + e % Wc;
            } else {                               // ghost columns (x sides), the other rows
                const int e2 = e - gr * Wc, k = e2 % max(gc, 1);
                jj = max(r0, 2) + e2 / max(gc, 1);
                ii = k < clo ? c0 + k : max(c0, nx + 2) + (k - clo);
            }
            bool xn, yn;
            const int si = phys_src(ii, nx, a.phys_bc[0], a.phys_bc[1], xn);
            const int sj = phys_src(jj, ny, a.phys_bc[2], a.phys_bc[3], yn);
            const bool ok = e < G;
            const int64_t src = ok ? (int64_t)(si + 2) * p.pitch + (sj + 2) : 0;
            dst[u] = ok ? (int64_t)ii * p.pitch + jj : -1;
            neg[u] = (xn ? 1u << nnx : 0u) ^ (yn ? 1u << nny : 0u);
#pragma unroll
            for (int c = 0; c < 3; ++c) v[u][c] = __ldcg(q + c * cs + src);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (dst[u] < 0) continue;
#pragma unroll
            for (int c = 0; c < 3; ++c) q[c * cs + dst[u]] = (neg[u] >> c) & 1u ? -v[u][c] : v[u][c];
        }
    }
}

template <int SYS, int FORM, bool REV, int LIM, bool CFL, bool RST = false, bool PFILL = false, bool SQ = false,
          bool WD = false, bool HM = false>
#ifdef K1_MAXREG
__global__ void __maxnreg__(K1_MAXREG) k1_fast(AdjStepArgs a) {
#else
__global__ void __launch_bounds__(32 * K1_WARPS, HM ? K1_MIN_BLOCKS_HM : K1_MIN_BLOCKS) k1_fast(AdjStepArgs a) {
#endif
    const int lane = threadIdx.x & 31;
    __shared__ int s_tile[K1_WARPS];
    constexpr int NARR = Strip<SYS, FORM, REV, LIM, CFL, RST, SQ, WD, false>::NARR;   // HM: room for the per-cell march
    extern __shared__ __align__(16) double s_ring1[];   // [K1_WARPS][RING1 * NARR * 32]
    const int warp = threadIdx.x >> 5;
#if K1_BULK
    __shared__ __align__(8) unsigned long long s_mbar[K1_WARPS][NGRP];
    unsigned bulk_phase = 0;
    if (lane == 0) {
        for (int gI = 0; gI < NGRP; ++gI)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&s_mbar[warp][gI])) : "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    __syncwarp();
#endif
    const int njob = a.job_offsets ? a.njob : a.ntile;
    // Each warp's first job is its warp index (no queue round trip); the job
    // tables are static, so its strip's table entries load before the wait for
    // the previous launch (PDL) -- a one-wave level (small AMR patches) keeps
    // that latency off its critical path.  Later jobs come from the queue.
    // (levels of small patches; a patch spanning its level -- PFILL -- keeps the queue for every job)
    constexpr bool SF = K1_STATIC_FIRST && !PFILL;
    const int total = SF ? gridDim.x * K1_WARPS : 0;
    int job0 = blockIdx.x * K1_WARPS + warp;
    int t0f = job0, t1f = job0 + 1;
    if (SF && job0 < njob && a.job_offsets) { t0f = a.job_offsets[job0]; t1f = a.job_offsets[job0 + 1]; }
    pdl_wait();
    pdl_trigger();
    if (!CFL && a.prefill.plan.n > 0) {      // the level's ghost fill, then every CTA waits for it
        prefill_gather(a.prefill);
        grid_barrier(a.work_counter + 2, gridDim.x);
    }
    for (bool first = SF;; first = false) {
        int job = job0, t0 = t0f, t1 = t1f;
        if (!first) {   // persistent warps: further strip jobs from a global queue until empty
            if (lane == 0) s_tile[warp] = total + atomicAdd(a.work_counter, 1);
            __syncwarp();
            job = s_tile[warp];
            __syncwarp();
            if (job < njob && a.job_offsets) { t0 = a.job_offsets[job]; t1 = a.job_offsets[job + 1]; }
            else { t0 = job; t1 = job + 1; }
        }
        if (job >= njob) {
            release_counter(a, lane, gridDim.x * K1_WARPS);
            break;
        }
        // this lane's strip: single-strip jobs use all lanes; packed jobs
        // stack up to four short strips (same ni) along the lanes
        int tix = t1 - 1, lane0 = a.job_offsets ? a.tiles[tix].pad : 0;
        for (int t = t0; t < t1 - 1; ++t) {
            const int next0 = a.tiles[t + 1].pad;
            if (lane < next0) { tix = t; lane0 = a.tiles[t].pad; break; }
        }
        if (!CFL && a.job_fill.n > 0) {   // this job's ghost cells, then every lane sees them
            job_fill(a.job_fill, const_cast<double*>(a.q_in), a.comp_stride, job, lane);
            __syncwarp();
        }
        if (PFILL) {   // the physical ghosts of every strip of this job, then the march reads them
            for (int t = t0; t < t1; ++t) {
                const AdjTile Tt = a.tiles[t];
                phys_prefill(a, Tt, a.patches[Tt.patch], lane);
            }
            __threadfence_block();
#if K1_BULK
            asm volatile("fence.proxy.async;\n" ::: "memory");   // the bulk copies read these generic stores
#endif
            __syncwarp();
        }
        const AdjTile T = a.tiles[tix];
        const AdjPatch p = a.patches[T.patch];
#if K1_BULK
        // a single strip on lanes 0..31 whose row segments are 16-byte aligned
        const bool bulk_ok = t1 - t0 == 1 && lane0 == 0 && ((p.offset + T.j0) & 1) == 0 && (p.pitch & 1) == 0 &&
                             (a.comp_stride & 1) == 0 && (a.aux_stride & 1) == 0;
        const unsigned bulk_bar = (unsigned)__cvta_generic_to_shared(&s_mbar[warp][0]);
#define K1_BULK_SET(S) (S).bulk = bulk_ok; (S).mbar = bulk_bar; (S).phase = &bulk_phase;
#else
#define K1_BULK_SET(S)
#endif
        if (WD && a.job_class) {   // wet/dry level: all-wet jobs march without the selects, all-dry ones copy
            const int cls = a.job_class[job];
            if (cls == 0) {
                Strip<SYS, FORM, REV, LIM, CFL, RST, SQ, false> S;
                S.smx = 0.0; S.smy = 0.0; S.bad = 0u;
                S.setup(T, p, a, lane, lane0, s_ring1 + warp * RING1 * NARR * 32);
                K1_BULK_SET(S)
                S.template run<1>();   // three columns per loop body here: the kernel also holds the wet/dry march
                if (S.bad) a.nonfinite[T.patch] = 1;
                continue;
            }
            if (cls == 2) {
                if (dry_copy(a, T, p, lane, lane0)) a.nonfinite[T.patch] = 1;
                continue;
            }
        }
        if (HM) {   // homogeneous level, or this job's strips read one material: the invariant march
            double hc = a.uniform_c, hz = a.uniform_z;
            if (a.job_uniform) { hc = __ldg(a.job_uniform + 2 * job); hz = __ldg(a.job_uniform + 2 * job + 1); }
            if (hc > 0.0) {
                Strip<SYS, FORM, REV, LIM, CFL, RST, SQ, WD, true> S;
                S.smx = 0.0; S.smy = 0.0; S.bad = 0u;
                S.setup(T, p, a, lane, lane0, s_ring1 + warp * RING1 * NARR * 32, hc, hz);
                K1_BULK_SET(S)
                S.run();
                if (S.bad) a.nonfinite[T.patch] = 1;
                continue;
            }
        }
        Strip<SYS, FORM, REV, LIM, CFL, RST, SQ, WD, false> S;
        S.smx = 0.0; S.smy = 0.0; S.bad = 0u;
        S.setup(T, p, a, lane, lane0, s_ring1 + warp * RING1 * NARR * 32);
        K1_BULK_SET(S)
        S.run();
        if (CFL) {   // single-strip jobs only (packed jobs require static_speed)
            const double smx = warp_max(S.smx), smy = warp_max(S.smy);
            if (lane == 0) {
                if (smx > 0.0) atomic_max_nonneg(&a.speed_max[2 * T.patch], smx);
                if (smy > 0.0) atomic_max_nonneg(&a.speed_max[2 * T.patch + 1], smy);
            }
        }
        if (S.bad) a.nonfinite[T.patch] = 1;
    }
}

// ---------------------------------------------------------------------------
// Two rows per lane: a warp owns 64 rows (60 outputs).  Lane l holds rows
// a = 2l and b = 2l+1 of the strip (relative to j0-2); the y-face between
// them is local, the one above b needs lane l+1's row a.  Each lane carries
// two independent dependency chains (more ILP at the same occupancy) and the
// shuffles per cell halve.  Used with the static CFL bound only.
template <int SYS, int FORM, bool REV, int LIM>
struct Strip2 {
    static constexpr bool SWE = SYS == ADJ_SYS_SWE2D;
    static constexpr int NARR = SWE ? 4 : 5;
    const double* __restrict__ qin[2];
    const double* __restrict__ aux[2];
    double* __restrict__ qout[2];
    int64_t cs, as;
    int pitch, g, ni, s_last, colbase;
    bool out[2];
    double dtdx, dtdy, hx, hy;
    double* ring;                  // [RING][NARR][64]
    int lane;

    Mat m[3][2];
    double q0[3][2], q1[3][2], q2[3][2];
    Face xf[3][2];
    double sy0[3][2], sy2[3][2];
    double gt0[3][2], gt2[3][2];   // gtil at the row's top face (row a: a|b, row b: b|a')
    double cy0[3][2], cy2[3][2];
    double bpy0[3][2], bpy1[3][2];
    double ft0[3][2], ft1[3][2];
    double sx0[3][2], sx1[3][2];
    double cup[3], mup[3];         // next lane's row a material (row above b)
    bool bad;

    ADJ_D void prefetch(int s, int slot) const {
        if (s <= s_last) {
            const int64_t o = (int64_t)(colbase + s) * pitch;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const double* src[5] = {qin[r] + o, qin[r] + cs + o, qin[r] + 2 * cs + o, aux[r] + o, aux[r] + as + o};
#pragma unroll
                for (int k = 0; k < NARR; ++k) {
                    const unsigned dst = (unsigned)__cvta_generic_to_shared(ring + (slot * NARR + k) * 64 + 2 * lane + r);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src[k]) : "memory");
                }
            }
        }
    }

    ADJ_D static void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

    ADJ_D void read(int slot, Raw& A, Raw& B) const {
        const double2* r = reinterpret_cast<const double2*>(ring + slot * NARR * 64) + lane;
        const double2 v0 = r[0], v1 = r[32], v2 = r[64], v3 = r[96];
        A.q0 = v0.x; B.q0 = v0.y; A.q1 = v1.x; B.q1 = v1.y; A.q2 = v2.x; B.q2 = v2.y; A.c = v3.x; B.c = v3.y;
        if (!SWE) { const double2 v4 = r[128]; A.z = v4.x; B.z = v4.y; } else { A.z = 0.0; B.z = 0.0; }
    }

    template <int K>
    ADJ_D void column(int s, const Raw& RA, const Raw& RB) {
        constexpr int C = K, P = (K + 2) % 3, PP = (K + 1) % 3;
        m[C][0] = make_mat<SYS, FORM, LIM>(RA.c, RA.z, dtdx, dtdy);
        m[C][1] = make_mat<SYS, FORM, LIM>(RB.c, RB.z, dtdx, dtdy);
        q0[C][0] = RA.q0; q1[C][0] = RA.q1; q2[C][0] = RA.q2;
        q0[C][1] = RB.q0; q1[C][1] = RB.q1; q2[C][1] = RB.q2;

        // ---- x-faces s-1/2, both rows
#pragma unroll
        for (int r = 0; r < 2; ++r)
            xf[C][r] = solve_face<SYS, FORM, REV>(q0[P][r], q1[P][r], q0[C][r], q1[C][r], m[P][r], m[C][r]);

        // ---- y-faces: F1 = a|b (local), F2 = b|a' (a' = next lane's row a)
        const Face F1 = solve_face<SYS, FORM, REV>(RA.q0, RA.q2, RB.q0, RB.q2, m[C][0], m[C][1]);
        const double uq0 = sh_dn(RA.q0), uq2 = sh_dn(RA.q2);
        Mat mu{};
        mu.c = sh_dn(m[C][0].c);
        mu.m = SWE ? mu.c : sh_dn(m[C][0].m);
        mu.k1 = fma(mu.m, mu.m, 1.0);
        mu.ky = sh_dn(m[C][0].ky);
        mu.tr = SWE ? mu.c * mu.c : mu.c * mu.m;
        mu.fx = FORM == ADJ_FORM_FWAVE ? sh_dn(m[C][0].fx) : 0.0;
        const Face F2 = solve_face<SYS, FORM, REV>(RB.q0, RB.q2, uq0, uq2, m[C][1], mu);
        {
            // F1: previous face = lane-1's F2, next face = own F2
            const double s0n = REV ? sh_up(F2.s0) : F2.s0;
            const double s1n = REV ? F2.s1 : sh_up(F2.s1);
            const double P0n = REV ? sh_up(F2.P) : 0.0;
            const double P1n = REV ? F2.P : 0.0;
            correction<SYS, FORM, REV, LIM>(F1, s0n, P0n, s1n, P1n, m[C][0], m[C][1], m[C][0].ky, m[C][1].ky,
                                            cy0[C][0], cy2[C][0]);
        }
        {
            // F2: previous face = own F1, next face = lane+1's F1
            const double s0n = REV ? F1.s0 : sh_dn(F1.s0);
            const double s1n = REV ? sh_dn(F1.s1) : F1.s1;
            const double P0n = REV ? F1.P : 0.0;
            const double P1n = REV ? sh_dn(F1.P) : 0.0;
            correction<SYS, FORM, REV, LIM>(F2, s0n, P0n, s1n, P1n, m[C][1], mu, m[C][1].ky, mu.ky,
                                            cy0[C][1], cy2[C][1]);
        }
        sy0[C][0] = F1.am0 + sh_up(F2.ap0);
        sy2[C][0] = F1.am1 + sh_up(F2.ap1);
        sy0[C][1] = F2.am0 + F1.ap0;
        sy2[C][1] = F2.am1 + F1.ap1;
        cup[C] = mu.c;
        mup[C] = mu.m;

        // ---- Sx(s-1) and its transverse split (rows above / below, column s-1)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            sx0[P][r] = xf[P][r].ap0 + xf[C][r].am0;
            sx1[P][r] = xf[P][r].ap1 + xf[C][r].am1;
        }
        {
            Mat mb{};                       // row a-1 = lane-1's row b
            mb.c = sh_up(m[P][1].c);
            mb.m = SWE ? mb.c : sh_up(m[P][1].m);
            mb.tr = SWE ? mb.c * mb.c : mb.c * mb.m;
            Mat ma{};                       // row b+1 = lane+1's row a
            ma.c = cup[P]; ma.m = mup[P];
            ma.tr = SWE ? ma.c * ma.c : ma.c * ma.m;
            double amA0, amAv, apA0, apAv, amB0, amBv, apB0, apBv;
            transverse<SYS, FORM, REV>(sx0[P][0], hx, mb, m[P][1], amA0, amAv, apA0, apAv);
            transverse<SYS, FORM, REV>(sx0[P][1], hx, m[P][0], ma, amB0, amBv, apB0, apBv);
            gt0[P][0] = cy0[P][0] - (apA0 - amB0);
            gt2[P][0] = cy2[P][0] - (apAv + amBv);
            gt0[P][1] = cy0[P][1] - (apB0 - sh_dn(amA0));
            gt2[P][1] = cy2[P][1] - (apBv + sh_dn(amAv));
        }

        // ---- transverse of Sy(s-1) with columns s-2, s; x-limiter of face s-3/2
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            double nbm0, bmv, bp0, bpv;
            transverse<SYS, FORM, REV>(sy0[P][r], hy, m[PP][r], m[C][r], nbm0, bmv, bp0, bpv);
            double fc0, fc1;
            correction<SYS, FORM, REV, LIM>(xf[P][r], REV ? xf[PP][r].s0 : xf[C][r].s0, xf[PP][r].P,
                                            REV ? xf[C][r].s1 : xf[PP][r].s1, xf[C][r].P,
                                            m[PP][r], m[P][r], m[PP][r].kx, m[P][r].kx, fc0, fc1);
            ft0[P][r] = fc0 - (bpy0[PP][r] - nbm0);
            ft1[P][r] = fc1 - (bpy1[PP][r] + bmv);
            bpy0[P][r] = bp0; bpy1[P][r] = bpv;
        }

        // ---- update cells of column s-2
        const double gb0 = sh_up(gt0[PP][1]), gb2 = sh_up(gt2[PP][1]);   // face below row a
        if (s >= 2 && s <= s_last) {
            const int64_t o = (int64_t)(colbase + s - 2) * pitch;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (!out[r]) continue;
                const double b0 = r == 0 ? gb0 : gt0[PP][0], b2 = r == 0 ? gb2 : gt2[PP][0];
                const double d0 = -dtdx * ((sx0[PP][r] + ft0[P][r]) - ft0[PP][r]) - dtdy * ((sy0[PP][r] + gt0[PP][r]) - b0);
                const double d1 = -dtdx * ((sx1[PP][r] + ft1[P][r]) - ft1[PP][r]);
                const double d2 = -dtdy * ((sy2[PP][r] + gt2[PP][r]) - b2);
                const double n0 = q0[PP][r] + d0, n1 = q1[PP][r] + d1, n2 = q2[PP][r] + d2;
                qout[r][o] = n0; qout[r][cs + o] = n1; qout[r][2 * cs + o] = n2;
                bad |= !(isfinite(n0) && isfinite(n1) && isfinite(n2));
            }
        }
    }

    ADJ_D void setup(const AdjTile& T, const AdjPatch& p, const AdjStepArgs& a, int lane_, double* ring_) {
        lane = lane_;
        ring = ring_;
        g = a.ghost;
        const int NY = p.ny + 2 * g;
        cs = a.comp_stride; as = a.aux_stride;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int l = 2 * lane + r;                 // row within the 64-row strip
            const int jj = g + T.j0 - 2 + l;
            const int jl = jj < 0 ? 0 : (jj > NY - 1 ? NY - 1 : jj);
            out[r] = l >= 2 && l < 2 + T.nj;
            qin[r] = a.q_in + p.offset + jl;
            aux[r] = a.aux + p.offset + jl;
            qout[r] = a.q_out + p.offset + jl;
        }
        pitch = p.pitch;
        dtdx = a.dtdx; dtdy = a.dtdy;
        hx = 0.5 * dtdx; hy = 0.5 * dtdy;
        colbase = g + T.i0;
        ni = T.ni;
    }

    ADJ_D void run() {
        const int s_first = -2;
        s_last = ni + 1;
        for (int gI = 0; gI < GROUPS; ++gI) {
            for (int k = 0; k < 3; ++k) prefetch(s_first + 3 * gI + k, 3 * gI + k);
            commit();
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                m[k][r] = Mat{}; xf[k][r] = Face{};
                q0[k][r] = q1[k][r] = q2[k][r] = 0.0;
                sy0[k][r] = sy2[k][r] = gt0[k][r] = gt2[k][r] = cy0[k][r] = cy2[k][r] = 0.0;
                bpy0[k][r] = bpy1[k][r] = ft0[k][r] = ft1[k][r] = sx0[k][r] = sx1[k][r] = 0.0;
            }
            cup[k] = mup[k] = 0.0;
        }
        int base = 0;
#pragma unroll 1
        for (int s = s_first; s <= s_last; s += 3) {
            asm volatile("cp.async.wait_group %0;\n" ::"n"(GROUPS - 1) : "memory");
            Raw a0, b0, a1, b1, a2, b2;
            read(base, a0, b0);
            read(base + 1, a1, b1);
            read(base + 2, a2, b2);
            prefetch(s + RING, base);
            prefetch(s + RING + 1, base + 1);
            prefetch(s + RING + 2, base + 2);
            commit();
            column<0>(s, a0, b0);
            column<1>(s + 1, a1, b1);
            column<2>(s + 2, a2, b2);
            base = base + 3 == RING ? 0 : base + 3;
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
    }
};

#ifndef K1_MIN_BLOCKS2
#define K1_MIN_BLOCKS2 2
#endif

template <int SYS, int FORM, bool REV, int LIM>
__global__ void __launch_bounds__(128, K1_MIN_BLOCKS2) k1_fast2(AdjStepArgs a) {
    const int lane = threadIdx.x & 31;
    __shared__ int s_tile[4];
    constexpr int NARR = Strip2<SYS, FORM, REV, LIM>::NARR;
    extern __shared__ __align__(16) double s_ring2[];            // [4 warps][RING][NARR][64]
    const int warp = threadIdx.x >> 5;
    pdl_wait();
    pdl_trigger();
    for (;;) {
        if (lane == 0) s_tile[warp] = atomicAdd(a.work_counter, 1);
        __syncwarp();
        const int job = s_tile[warp];
        __syncwarp();
        if (job >= a.ntile) {
            release_counter(a, lane, gridDim.x * 4);
            break;
        }
        const AdjTile T = a.tiles[job];
        const AdjPatch p = a.patches[T.patch];
        Strip2<SYS, FORM, REV, LIM> S;
        S.bad = false;
        S.setup(T, p, a, lane, s_ring2 + warp * RING * NARR * 64);
        S.run();
        if (S.bad) a.nonfinite[T.patch] = 1;
    }
}

template <int SYS, int FORM, bool REV, int LIM>
static void launch_two_rows(const AdjStepArgs& a, cudaStream_t st) {
    static int blocks_per_sm = 0, sms = 0;
    constexpr int smem = 4 * RING * Strip2<SYS, FORM, REV, LIM>::NARR * 64 * (int)sizeof(double);
    if (blocks_per_sm == 0) {
        cudaFuncSetAttribute(k1_fast2<SYS, FORM, REV, LIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k1_fast2<SYS, FORM, REV, LIM>, 128, smem);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    int blocks = blocks_per_sm * sms;
    const int need = (a.ntile + 3) / 4;
    if (blocks > need) blocks = need;
    launch_pdl(k1_fast2<SYS, FORM, REV, LIM>, dim3(blocks), dim3(128), smem, st, a);
}

template <int SYS, int FORM, bool REV, int LIM, bool CFL, bool RST = false, bool PFILL = false, bool SQ = false,
          bool WD = false, bool HM = false>
static void launch_cfl(const AdjStepArgs& a, cudaStream_t st) {
    static int blocks_per_sm = 0, sms = 0;
    constexpr int smem =
        K1_WARPS * RING1 * Strip<SYS, FORM, REV, LIM, CFL, RST, SQ, WD, false>::NARR * 32 * (int)sizeof(double);
    if (blocks_per_sm == 0) {
        cudaFuncSetAttribute(k1_fast<SYS, FORM, REV, LIM, CFL, RST, PFILL, SQ, WD, HM>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &blocks_per_sm, k1_fast<SYS, FORM, REV, LIM, CFL, RST, PFILL, SQ, WD, HM>, 32 * K1_WARPS, smem);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    int blocks = blocks_per_sm * sms;
    const int need = ((a.job_offsets ? a.njob : a.ntile) + K1_WARPS - 1) / K1_WARPS;
    if (blocks > need) blocks = need;
    launch_pdl(k1_fast<SYS, FORM, REV, LIM, CFL, RST, PFILL, SQ, WD, HM>, dim3(blocks), dim3(32 * K1_WARPS), smem, st, a);
}

// Square cells (dt/dx == dt/dy, every BASELINE configuration) share the x and
// y correction magnitudes: a separate instantiation (SQ) of the static-CFL
// kernels for the MC limiter drops their recomputation.
template <int SYS, int FORM, bool REV, int LIM, bool SQ>
static void launch_static(const AdjStepArgs& a, cudaStream_t st) {
    if constexpr (SYS == ADJ_SYS_AC2D && FORM == ADJ_FORM_WAVE && !REV) {   // homogeneous acoustics levels
        if (a.flags & ADJ_STEP_UNIFORM_MAT) {
            if (a.fine_restrict.ratio > 0) launch_cfl<SYS, FORM, REV, LIM, false, true, false, SQ, false, true>(a, st);
            else if (a.flags & ADJ_STEP_PHYS_IN) launch_cfl<SYS, FORM, REV, LIM, false, false, true, SQ, false, true>(a, st);
            else launch_cfl<SYS, FORM, REV, LIM, false, false, false, SQ, false, true>(a, st);
            return;
        }
    }
    if constexpr (FORM == ADJ_FORM_WAVE && !REV) {   // forward levels: optional fused restriction
        if (a.fine_restrict.ratio > 0) {
            launch_cfl<SYS, FORM, REV, LIM, false, true, false, SQ>(a, st);
            return;
        }
    }
    if (a.flags & ADJ_STEP_PHYS_IN) launch_cfl<SYS, FORM, REV, LIM, false, false, true, SQ>(a, st);
    else launch_cfl<SYS, FORM, REV, LIM, false, false, false, SQ>(a, st);
}

// Shallow water with dry cells (ADJ_STEP_WET_DRY): forward wave form or the
// time-reversed f-wave adjoint, static CFL bound, no fused restriction
// (shallow water restricts wet-weighted); step_fast checks the arguments.
template <int SYS, int FORM, bool REV, int LIM>
static void launch_wet_dry(const AdjStepArgs& a, cudaStream_t st) {
    if constexpr (SYS == ADJ_SYS_SWE2D && ((FORM == ADJ_FORM_WAVE && !REV) || (FORM == ADJ_FORM_FWAVE && REV))) {
        const bool pin = a.flags & ADJ_STEP_PHYS_IN;
        if constexpr (LIM == ADJ_LIM_MC) {
            if (a.dtdx == a.dtdy) {
                if (pin) launch_cfl<SYS, FORM, REV, LIM, false, false, true, true, true>(a, st);
                else launch_cfl<SYS, FORM, REV, LIM, false, false, false, true, true>(a, st);
                return;
            }
        }
        if (pin) launch_cfl<SYS, FORM, REV, LIM, false, false, true, false, true>(a, st);
        else launch_cfl<SYS, FORM, REV, LIM, false, false, false, false, true>(a, st);
    }
}

template <int SYS, int FORM, bool REV, int LIM>
static void launch_kernel(const AdjStepArgs& a, cudaStream_t st) {
    if (a.flags & ADJ_STEP_WET_DRY) {
        launch_wet_dry<SYS, FORM, REV, LIM>(a, st);
        return;
    }
    if ((a.flags & ADJ_STEP_TWO_ROWS) && a.static_speed && !a.job_offsets && !(a.flags & ADJ_STEP_PHYS_IN) &&
        !(FORM == ADJ_FORM_WAVE && !REV && a.fine_restrict.ratio > 0)) {
        launch_two_rows<SYS, FORM, REV, LIM>(a, st);
    } else if (a.static_speed) {
        if constexpr (LIM == ADJ_LIM_MC) {
            if (a.dtdx == a.dtdy) {
                launch_static<SYS, FORM, REV, LIM, true>(a, st);
                return;
            }
        }
        launch_static<SYS, FORM, REV, LIM, false>(a, st);
    } else if (!a.job_offsets) {
        launch_cfl<SYS, FORM, REV, LIM, true>(a, st);
    }
}

template <int SYS, int FORM, bool REV>
static void launch_lim(const AdjStepArgs& a, cudaStream_t st) {
    switch (a.limiter) {
        case ADJ_LIM_NONE: launch_kernel<SYS, FORM, REV, ADJ_LIM_NONE>(a, st); break;
        case ADJ_LIM_MINMOD: launch_kernel<SYS, FORM, REV, ADJ_LIM_MINMOD>(a, st); break;
        case ADJ_LIM_MC: launch_kernel<SYS, FORM, REV, ADJ_LIM_MC>(a, st); break;
        default: launch_kernel<SYS, FORM, REV, ADJ_LIM_SUPERBEE>(a, st); break;
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
    if (a.job_offsets && !a.static_speed) return ADJ_ERR_BAD_ARG;   // packed jobs need the static CFL bound
    if ((a.flags & ADJ_STEP_WET_DRY) &&
        !(a.system == ADJ_SYS_SWE2D && a.static_speed && a.fine_restrict.ratio <= 0 &&
          ((a.form == ADJ_FORM_WAVE && !a.reversed) || (a.form == ADJ_FORM_FWAVE && a.reversed))))
        return ADJ_ERR_BAD_ARG;   // dry cells: shallow water forward (wave) or adjoint (time-reversed f-wave),
                                  // static CFL bound, no fused restriction
    if (a.system == ADJ_SYS_AC2D) fast::launch_sys<ADJ_SYS_AC2D>(a, st);
    else if (a.system == ADJ_SYS_SWE2D) fast::launch_sys<ADJ_SYS_SWE2D>(a, st);
    else return ADJ_ERR_BAD_ARG;
    return check_launch("k1_fast");
}

}  // namespace adj
