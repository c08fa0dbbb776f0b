// K2 ghost fill and K4 restriction.  Compiled with -fmad=false: every value
// is produced with the reference's operation order, so results are bitwise
// identical to the numpy reference.
//
//   fill_ghost_physical + _mirror/_extrapolate  solver.py:84-146
//   fill_ghost_same_level                       solver.py:208-224
//   fill_ghost_from_coarse / space_time_interp  solver.py:227-286
//   interpolate_patch / _axis_weights           geometry.py:248-260, 302-327
//   restrict_fine_to_coarse                     amr.py:399-450
#include "adj_common.cuh"
#include <stdlib.h>

namespace adj {

// ---------------------------------------------------------------------------
// Physical boundaries.  The reference fills whole slabs x-low, x-high, y-low,
// y-high in that order; because every slab source row is interior, the final
// value of any out-of-domain ghost cell is the composition
//   q[c](ii,jj) = sy_c * sx_c * q_pre[c](src_x(ii), src_y(jj))
// which one gather computes without a second pass.
ADJ_D int phys_src(int ii, int n, int g, bool lo_edge, bool hi_edge, int bc_lo, int bc_hi,
                   bool* neg, bool* hit) {
    *neg = false; *hit = false;
    if (ii < g && lo_edge) {
        *hit = true;
        if (bc_lo == ADJ_BC_WALL) { *neg = true; return 2 * g - 1 - ii; }
        if (bc_lo == ADJ_BC_PERIODIC) return ii + n - 2 * g;   // the patch spans the axis
        return g;
    }
    if (ii >= n - g && hi_edge) {
        *hit = true;
        if (bc_hi == ADJ_BC_WALL) { *neg = true; return 2 * n - 2 * g - 1 - ii; }
        if (bc_hi == ADJ_BC_PERIODIC) return ii - (n - 2 * g);
        return n - g - 1;
    }
    return ii;
}

__global__ void k2_physical(AdjPhysArgs a) {
    pdl_wait();
    pdl_trigger();
    const AdjPatch p = a.patches[blockIdx.y];
    const int g = a.ghost;
    const int NX = p.nx + 2 * g;
    const int gy = a.ndim == 2 ? g : 0;
    const int NY = p.ny + 2 * gy;
    const int64_t ring = (int64_t)NX * NY - (int64_t)p.nx * p.ny;
    const bool xlo = p.edges & ADJ_EDGE_XLO, xhi = p.edges & ADJ_EDGE_XHI;
    const bool ylo = a.ndim == 2 && (p.edges & ADJ_EDGE_YLO), yhi = a.ndim == 2 && (p.edges & ADJ_EDGE_YHI);
    if (!(xlo || xhi || ylo || yhi)) return;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < ring;
         r += (int64_t)gridDim.x * blockDim.x) {
        int ii, jj;
        const int64_t band = (int64_t)g * NY;
        if (r < band) { ii = (int)(r / NY); jj = (int)(r % NY); }
        else if (r < 2 * band) { int64_t s = r - band; ii = NX - g + (int)(s / NY); jj = (int)(s % NY); }
        else {
            int64_t s = r - 2 * band;             // middle rows, 2*gy cells each
            ii = g + (int)(s / (2 * gy));
            int k = (int)(s % (2 * gy));
            jj = k < gy ? k : NY - 2 * gy + k;
        }
        bool nx_, hx, ny_, hy;
        int sx = phys_src(ii, NX, g, xlo, xhi, a.bc[0], a.bc[1], &nx_, &hx);
        int sy = jj;
        ny_ = false; hy = false;
        if (a.ndim == 2) sy = phys_src(jj, NY, g, ylo, yhi, a.bc[2], a.bc[3], &ny_, &hy);
        if (!hx && !hy) continue;
        const int64_t dst = p.offset + (int64_t)ii * p.pitch + jj;
        const int64_t src = p.offset + (int64_t)sx * p.pitch + sy;
        for (int c = 0; c < a.m; ++c) {
            double v = a.q[c * a.comp_stride + src];
            if (nx_ && c == a.normal_comp[0]) v = v * -1.0;
            if (ny_ && c == a.normal_comp[1]) v = v * -1.0;
            a.q[c * a.comp_stride + dst] = v;
        }
    }
}

int fill_physical(const AdjPhysArgs& a) {
    if (a.npatch <= 0 || a.max_ghost_cells <= 0) return ADJ_OK;
    int blocks = (a.max_ghost_cells + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    launch_pdl(k2_physical, dim3(blocks, a.npatch), dim3(256), 0, (cudaStream_t)a.stream, a);
    return check_launch("k2_physical");
}

// ---------------------------------------------------------------------------
// Same-level copies and coarse-to-fine space-time interpolation.

// _axis_weights (geometry.py:248-260) for one coordinate.
ADJ_D void axis_weights(double coord, double origin, double width, int n, int* i0, double* w) {
    double s = (coord - origin) / width - 0.5;
    double fl = floor(s);
    int k = (int)fl;
    double ww = s - fl;
    if (k < 0) ww = 0.0;
    else if (k > n - 2) ww = 1.0;
    int hi = n - 2 > 0 ? n - 2 : 0;
    k = k < 0 ? 0 : (k > hi ? hi : k);
    if (n == 1) ww = 0.0;
    *i0 = k;
    *w = ww;
}

// interpolate_patch (geometry.py:302-327) for one point and component.
ADJ_D double interp_patch2(const double* d, int pitch, int i0, int j0, int i1, int j1, double wx, double wy) {
    double v00 = d[(int64_t)i0 * pitch + j0], v10 = d[(int64_t)i1 * pitch + j0];
    double v01 = d[(int64_t)i0 * pitch + j1], v11 = d[(int64_t)i1 * pitch + j1];
    return v00 * (1.0 - wx) * (1.0 - wy) + v10 * wx * (1.0 - wy) + v01 * (1.0 - wx) * wy + v11 * wx * wy;
}

// One warp per rectangle, RECTS_PER_CTA warps per CTA (ghost rectangles are
// small: 2 x 32 cells for a 32^2 patch side).
constexpr int RECTS_PER_CTA = 8;

__global__ void __launch_bounds__(32 * RECTS_PER_CTA) k2_rects(AdjGhostArgs a) {
    const int rid = blockIdx.x * RECTS_PER_CTA + (threadIdx.x >> 5);
    if (rid >= a.nrect) return;
    const int lane = threadIdx.x & 31;
    const AdjRect R = a.rects[rid];
    const AdjPatch dp = a.dst_patches[R.dst_patch];
    const AdjPatch sp = R.kind == ADJ_RECT_COPY ? a.src_patches[R.src_patch] : a.coarse_patches[R.src_patch];
    const int64_t n = (int64_t)R.ni * R.nj;
    for (int64_t t = lane; t < n; t += 32) {
        const int di = (int)(t / R.nj), dj = (int)(t % R.nj);
        const int ii = R.di0 + di, jj = R.dj0 + dj;
        const int64_t dst = dp.offset + (int64_t)ii * dp.pitch + jj;
        if (R.kind == ADJ_RECT_COPY) {
            const int64_t src = sp.offset + (int64_t)(R.si0 + di) * sp.pitch + (R.sj0 + dj);
            for (int c = 0; c < a.m; ++c)
                a.q_dst[c * a.dst_comp_stride + dst] = a.q_src[c * a.src_comp_stride + src];
            continue;
        }
        // COARSE: fine cell centre -> bilinear weights on the coarse patch incl. ghosts
        const int gc = a.ghost_src;
        const int ncx = sp.nx + 2 * gc;
        int i0, j0 = 0, j1 = 0;
        double wx, wy = 0.0;
        if (a.axis_w) {            // host-precomputed (same arithmetic, per rect row / column)
            i0 = a.axis_i[R.pad + di];
            wx = a.axis_w[R.pad + di];
            if (a.ndim == 2) {
                j0 = a.axis_i[R.pad + R.ni + dj];
                wy = a.axis_w[R.pad + R.ni + dj];
            }
        } else {
            const int gf = a.ghost_dst;
            const int gxi = dp.lo_x - gf + ii;
            const double x = a.origin_x + (gxi + 0.5) * a.dx_f;
            const double lox = a.origin_x + (sp.lo_x - gc) * a.dx_c;
            axis_weights(x, lox, a.dx_c, ncx, &i0, &wx);
            if (a.ndim == 2) {
                const int gyi = dp.lo_y - gf + jj;
                const double y = a.origin_y + (gyi + 0.5) * a.dy_f;
                const double loy = a.origin_y + (sp.lo_y - gc) * a.dy_c;
                axis_weights(y, loy, a.dy_c, sp.ny + 2 * gc, &j0, &wy);
            }
        }
        const int i1 = min(i0 + 1, ncx - 1);
        if (a.ndim == 2) j1 = min(j0 + 1, sp.ny + 2 * gc - 1);
        // graph replays read the weight from device memory; a negative value
        // there means "old state only" (w == 0 or t1 == t0, solver.py:280-284)
        double wt = a.w_time;
        int tmode = a.time_mode;
        if (a.w_time_dev) {
            wt = *a.w_time_dev;
            tmode = wt < 0.0 ? 0 : 1;
        }
        for (int c = 0; c < a.m; ++c) {
            double vo = 0.0, vn = 0.0;
            const double* po = a.q_coarse_old + c * a.coarse_comp_stride + sp.offset;
            const double* pn = a.q_coarse_new + c * a.coarse_comp_stride + sp.offset;
            if (a.ndim == 2) {
                if (tmode != 2) vo = interp_patch2(po, sp.pitch, i0, j0, i1, j1, wx, wy);
                if (tmode != 0) vn = interp_patch2(pn, sp.pitch, i0, j0, i1, j1, wx, wy);
            } else {
                if (tmode != 2) vo = po[i0] * (1.0 - wx) + po[i1] * wx;
                if (tmode != 0) vn = pn[i0] * (1.0 - wx) + pn[i1] * wx;
            }
            double v;
            if (tmode == 0) v = vo;
            else if (tmode == 2) v = vn;
            else v = (1.0 - wt) * vo + wt * vn;
            a.q_dst[c * a.dst_comp_stride + dst] = v;
        }
    }
}

int fill_ghost_rects(const AdjGhostArgs& a) {
    if (a.nrect <= 0) return ADJ_OK;
    const int blocks = (a.nrect + RECTS_PER_CTA - 1) / RECTS_PER_CTA;
    k2_rects<<<blocks, 32 * RECTS_PER_CTA, 0, (cudaStream_t)a.stream>>>(a);
    return check_launch("k2_rects");
}

// ---------------------------------------------------------------------------
// Planned level fill.  Build (once per regrid): one entry per ghost cell the
// fill writes, rect cells first (COARSE rects, then COPY rects, at the
// caller's prefix offsets), then the physical cells, each resolved to the
// entry or interior cell its composite source reads.  Fill: a flat gather.

__global__ void __launch_bounds__(32 * RECTS_PER_CTA) k2_plan_rects(AdjGhostPlanBuildArgs a) {
    const int rid = blockIdx.x * RECTS_PER_CTA + (threadIdx.x >> 5);
    if (rid >= a.nrect) return;
    const int lane = threadIdx.x & 31;
    const AdjRect R = a.rects[rid];
    const AdjPatch dp = a.patches[R.dst_patch];
    const bool coarse = R.kind == ADJ_RECT_COARSE;
    const AdjPatch sp = coarse ? a.coarse_patches[R.src_patch] : a.patches[R.src_patch];
    const int base = a.rect_cell0[rid];
    const int n = R.ni * R.nj;
    for (int t = lane; t < n; t += 32) {
        const int di = t / R.nj, dj = t - di * R.nj;
        const int pos = base + t;
        const int dst = (int)(dp.offset + (int64_t)(R.di0 + di) * dp.pitch + (R.dj0 + dj));
        a.plan.dst[pos] = dst;
        if (coarse) {
            const int gc = a.ghost_coarse;
            const int ncx = sp.nx + 2 * gc;
            const int i0 = a.axis_i[R.pad + di];
            int j0 = 0, j1 = 0;
            double wy = 0.0;
            if (a.ndim == 2) {
                j0 = a.axis_i[R.pad + R.ni + dj];
                wy = a.axis_w[R.pad + R.ni + dj];
                j1 = min(j0 + 1, sp.ny + 2 * gc - 1);
            }
            const int i1 = min(i0 + 1, ncx - 1);
            a.plan.c_base[pos] = (int)(sp.offset + (int64_t)i0 * sp.pitch + j0);
            a.plan.c_step[pos] = (i1 - i0) * sp.pitch | ((j1 - j0) << 30);
            a.plan.c_wx[pos] = a.axis_w[R.pad + di];
            a.plan.c_wy[pos] = wy;
            a.plan.src[pos] = pos;
            a.plan.meta[pos] = 1u;
        } else {
            a.plan.src[pos] = (int)(sp.offset + (int64_t)(R.si0 + di) * sp.pitch + (R.sj0 + dj));
            a.plan.meta[pos] = 0u;
        }
        if (a.owner) a.owner[dst] = pos;
    }
}

__global__ void k2_plan_physical(AdjGhostPlanBuildArgs a, int first) {
    const AdjPatch p = a.edge_patches[blockIdx.y];
    const int g = a.ghost;
    const int NX = p.nx + 2 * g;
    const int gy = a.ndim == 2 ? g : 0;
    const int NY = p.ny + 2 * gy;
    const int ring = NX * NY - p.nx * p.ny;
    const bool xlo = p.edges & ADJ_EDGE_XLO, xhi = p.edges & ADJ_EDGE_XHI;
    const bool ylo = a.ndim == 2 && (p.edges & ADJ_EDGE_YLO), yhi = a.ndim == 2 && (p.edges & ADJ_EDGE_YHI);
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ring; r += gridDim.x * blockDim.x) {
        int ii, jj;
        const int band = g * NY;
        if (r < band) { ii = r / NY; jj = r % NY; }
        else if (r < 2 * band) { const int s = r - band; ii = NX - g + s / NY; jj = s % NY; }
        else {
            const int s = r - 2 * band;
            ii = g + s / (2 * gy);
            const int k = s % (2 * gy);
            jj = k < gy ? k : NY - 2 * gy + k;
        }
        bool nx_, hx, ny_ = false, hy = false;
        const int sx = phys_src(ii, NX, g, xlo, xhi, a.bc[0], a.bc[1], &nx_, &hx);
        int sy = jj;
        if (a.ndim == 2) sy = phys_src(jj, NY, g, ylo, yhi, a.bc[2], a.bc[3], &ny_, &hy);
        if (!hx && !hy) continue;
        unsigned sign = 0u;
        if (nx_ && a.normal_comp[0] >= 0) sign ^= 2u << a.normal_comp[0];
        if (ny_ && a.normal_comp[1] >= 0) sign ^= 2u << a.normal_comp[1];
        const int dst = (int)(p.offset + (int64_t)ii * p.pitch + jj);
        const int src = (int)(p.offset + (int64_t)sx * p.pitch + sy);
        const int pos = first + atomicAdd(a.counter, 1);
        const int o = a.owner ? a.owner[src] : -1;
        a.plan.dst[pos] = dst;
        if (o >= 0) {               // source is a ghost the in-domain phases write
            a.plan.src[pos] = a.plan.src[o];
            a.plan.meta[pos] = a.plan.meta[o] ^ sign;
        } else {                    // interior (or untouched) cell of the same patch
            a.plan.src[pos] = src;
            a.plan.meta[pos] = sign;
        }
    }
}

int ghost_plan_build(const AdjGhostPlanBuildArgs& a, int rect_cells) {
    cudaStream_t st = (cudaStream_t)a.stream;
    if (a.nrect > 0) {
        const int blocks = (a.nrect + RECTS_PER_CTA - 1) / RECTS_PER_CTA;
        k2_plan_rects<<<blocks, 32 * RECTS_PER_CTA, 0, st>>>(a);
        int rc = check_launch("k2_plan_rects");
        if (rc) return rc;
    }
    if (a.nedge > 0 && a.max_ghost_cells > 0) {
        int bx = (a.max_ghost_cells + 255) / 256;
        if (bx > 4096) bx = 4096;
        k2_plan_physical<<<dim3(bx, a.nedge), 256, 0, st>>>(a, rect_cells);
        return check_launch("k2_plan_physical");
    }
    return ADJ_OK;
}

// interpolate_patch (geometry.py:302-327) / linear in 1D, reference order,
// at (i0, j0) with row step di and column step dj
template <int NDIM>
ADJ_D double interp_at(const double* p, int di, int dj, double wx, double wy) {
    if (NDIM == 2)
        return p[0] * (1.0 - wx) * (1.0 - wy) + p[di] * wx * (1.0 - wy) + p[dj] * (1.0 - wx) * wy +
               p[di + dj] * wx * wy;
    return p[0] * (1.0 - wx) + p[di] * wx;
}

#ifndef K2_GATHER_MINB
#define K2_GATHER_MINB 1   // resident CTAs per SM the gather's register budget targets (experiments)
#endif
template <int NDIM, int M, int U>
__global__ void __launch_bounds__(256, K2_GATHER_MINB) k2_gather(AdjGhostPlanFillArgs a) {
    pdl_wait();
    pdl_trigger();
    double wt = a.w_time;
    int tmode = a.time_mode;
    if (a.w_time_dev) {           // graph replays: negative weight = old state only
        wt = *a.w_time_dev;
        tmode = wt < 0.0 ? 0 : 1;
    }
    const int64_t cs = a.comp_stride, ccs = a.coarse_comp_stride;
    const int n = a.plan.n, nc = a.plan.nc;
    const int stride = gridDim.x * blockDim.x;
    // U entries per thread with all their loads issued before any use
    for (int t0 = blockIdx.x * blockDim.x + threadIdx.x; t0 < n; t0 += U * stride) {
        int dst[U], src[U], cb[U], step[U];
        unsigned meta[U];
        double wx[U], wy[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + u * stride;
            const bool ok = t < n;
            const int tt = ok ? t : 0;
            dst[u] = ok ? a.plan.dst[tt] : -1;
            src[u] = a.plan.src[tt];
            meta[u] = ok ? a.plan.meta[tt] : 0u;
            // rect COARSE entries [0, nc) own coarse entry t: load it alongside the plan entry
            const int ci = tt < nc ? tt : 0;
            cb[u] = nc ? a.plan.c_base[ci] : 0;
            step[u] = nc ? a.plan.c_step[ci] : 0;
            wx[u] = nc ? a.plan.c_wx[ci] : 0.0;
            wy[u] = nc ? a.plan.c_wy[ci] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if ((meta[u] & 1u) && t0 + u * stride >= nc) {   // physical cell mirroring a coarse-interpolated ghost
                const int c0 = src[u];
                cb[u] = a.plan.c_base[c0]; step[u] = a.plan.c_step[c0];
                wx[u] = a.plan.c_wx[c0]; wy[u] = a.plan.c_wy[c0];
            }
        }
        double v[U][M];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (meta[u] & 1u) {
                const int di = step[u] & 0x3fffffff, dj = (int)((unsigned)step[u] >> 30);
#pragma unroll
                for (int c = 0; c < M; ++c) {
                    const double* po = a.q_coarse_old + c * ccs + cb[u];
                    const double* pn = a.q_coarse_new + c * ccs + cb[u];
                    const double vo = tmode != 2 ? interp_at<NDIM>(po, di, dj, wx[u], wy[u]) : 0.0;
                    const double vn = tmode != 0 ? interp_at<NDIM>(pn, di, dj, wx[u], wy[u]) : 0.0;
                    v[u][c] = tmode == 0 ? vo : (tmode == 2 ? vn : (1.0 - wt) * vo + wt * vn);
                }
            } else {
#pragma unroll
                for (int c = 0; c < M; ++c) v[u][c] = dst[u] >= 0 ? a.q[c * cs + src[u]] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (dst[u] < 0) continue;
#pragma unroll
            for (int c = 0; c < M; ++c) a.q[c * cs + dst[u]] = (meta[u] >> (1 + c)) & 1u ? v[u][c] * -1.0 : v[u][c];
        }
    }
}

static int gather_batch() {
    static int u = -1;
    if (u < 0) {
        const char* e = getenv("ADJAMR_GATHER_U");
        u = (e && (e[0] == '1' || e[0] == '2' || e[0] == '4')) ? e[0] - '0' : 2;   // 2: measured best on C5
    }
    return u;
}

template <int NDIM, int M>
static void launch_gather(const AdjGhostPlanFillArgs& a, cudaStream_t st) {
    const int U = gather_batch();
    int blocks = (a.plan.n + 256 * U - 1) / (256 * U);
    if (blocks > 148 * 8) blocks = 148 * 8;
    const dim3 g(blocks), b(256);
    if (U == 4) launch_pdl(k2_gather<NDIM, M, 4>, g, b, 0, st, a);
    else if (U == 2) launch_pdl(k2_gather<NDIM, M, 2>, g, b, 0, st, a);
    else launch_pdl(k2_gather<NDIM, M, 1>, g, b, 0, st, a);
}

int fill_ghost_plan(const AdjGhostPlanFillArgs& a) {
    if (a.plan.n <= 0) return ADJ_OK;
    const cudaStream_t st = (cudaStream_t)a.stream;
    if (a.ndim == 2 && a.m == 3) launch_gather<2, 3>(a, st);
    else if (a.ndim == 1 && a.m == 2) launch_gather<1, 2>(a, st);
    else if (a.ndim == 2 && a.m == 2) launch_gather<2, 2>(a, st);
    else if (a.ndim == 1 && a.m == 3) launch_gather<1, 3>(a, st);
    else if (a.ndim == 1 && a.m == 1) launch_gather<1, 1>(a, st);
    else if (a.ndim == 2 && a.m == 1) launch_gather<2, 1>(a, st);
    else return ADJ_ERR_BAD_ARG;
    return check_launch("k2_gather");
}

// ---------------------------------------------------------------------------
// K4 restriction.  numpy's mean over the (r, r) child block (amr.py:440-450)
// sums each child row sequentially and adds the row sums in order, then
// divides by r*r -- except when the coarse box is one cell wide in y: numpy
// then reduces the r*r block as one flat row-major run with its pairwise
// summation (8 partial sums once n >= 8).  Both orders are reproduced so the
// result is bitwise equal; the SWE variant weights by the wet mask.
ADJ_D double block_sum(const double* f, const double* wet, int64_t pitch, int fi0, int fj0, int r, int rj,
                       bool flat) {
    auto val = [&](int p, int q) {
        const int64_t o = (int64_t)(fi0 + p) * pitch + fj0 + q;
        return wet ? f[o] * (wet[o] > 0.0 ? 1.0 : 0.0) : f[o];
    };
    if (flat) {
        const int n = r * rj;
        if (n < 8) {
            double s = val(0, 0);
            for (int e = 1; e < n; ++e) s = s + val(e / rj, e % rj);
            return s;
        }
        double acc[8];
        for (int e = 0; e < 8; ++e) acc[e] = val(e / rj, e % rj);
        int e = 8;
        for (; e + 8 <= n; e += 8)
            for (int j = 0; j < 8; ++j) acc[j] = acc[j] + val((e + j) / rj, (e + j) % rj);
        double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        for (; e < n; ++e) s = s + val(e / rj, e % rj);
        return s;
    }
    double tot = 0.0;
    for (int p = 0; p < r; ++p) {
        double s = val(p, 0);
        for (int q = 1; q < rj; ++q) s = s + val(p, q);
        tot = p == 0 ? s : tot + s;
    }
    return tot;
}

__global__ void k4_restrict(AdjRestrictArgs a) {
    pdl_wait();
    pdl_trigger();
    const AdjRect R = a.rects[blockIdx.x];
    const AdjPatch cp = a.coarse_patches[R.dst_patch];
    const AdjPatch fp = a.fine_patches[R.src_patch];
    const int r = a.ratio;
    const int rj = a.ndim == 2 ? r : 1;
    const bool flat = a.ndim == 2 && R.nj == 1;
    const int64_t n = (int64_t)R.ni * R.nj;
    const int gC = a.ghost_coarse, gF = a.ghost_fine;   // rect coords are interior-local
    for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
        const int di = (int)(t / R.nj), dj = (int)(t % R.nj);
        const int ci = gC + R.di0 + di;
        const int cj = (a.ndim == 2 ? gC : 0) + R.dj0 + dj;
        const int fi0 = gF + R.si0 + di * r;
        const int fj0 = (a.ndim == 2 ? gF : 0) + R.sj0 + dj * rj;
        const int64_t cdst = cp.offset + (int64_t)ci * cp.pitch + cj;
        if (!a.swe) {
            const double cnt = (double)(r * rj);
            for (int c = 0; c < a.m; ++c) {
                const double* f = a.q_fine + c * a.fine_comp_stride + fp.offset;
                a.q_coarse[c * a.coarse_comp_stride + cdst] = block_sum(f, nullptr, fp.pitch, fi0, fj0, r, rj, flat) / cnt;
            }
        } else {
            const double* fd = a.aux_fine + a.fine_aux_stride + fp.offset;   // depth plane
            double ws = 0.0;
            for (int p = 0; p < r; ++p)
                for (int q = 0; q < rj; ++q)
                    ws = ws + (fd[(int64_t)(fi0 + p) * fp.pitch + fj0 + q] > 0.0 ? 1.0 : 0.0);
            const bool wetc = a.aux_coarse[a.coarse_aux_stride + cp.offset + (int64_t)ci * cp.pitch + cj] > 0.0;
            if (!(ws > 0.0 && wetc)) continue;
            for (int c = 0; c < a.m; ++c) {
                const double* f = a.q_fine + c * a.fine_comp_stride + fp.offset;
                a.q_coarse[c * a.coarse_comp_stride + cdst] = block_sum(f, fd, fp.pitch, fi0, fj0, r, rj, flat) / ws;
            }
        }
    }
}

// Planned form: one thread per covered coarse cell, no rect / patch lookups.
template <int M, bool SWE>
__global__ void __launch_bounds__(256) k4_cells(AdjRestrictArgs a) {
    pdl_wait();
    pdl_trigger();
    const int r = a.ratio;
    const int rj = a.ndim == 2 ? r : 1;
    const double cnt = (double)(r * rj);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < a.ncell; t += gridDim.x * blockDim.x) {
        const int cdst = a.cell_dst[t], fsrc = a.cell_src[t], meta = a.cell_meta[t];
        const bool flat = meta & 1;
        const int fpitch = meta >> 1;
        if (!SWE) {
#pragma unroll
            for (int c = 0; c < M; ++c)
                a.q_coarse[c * a.coarse_comp_stride + cdst] =
                    block_sum(a.q_fine + c * a.fine_comp_stride + fsrc, nullptr, fpitch, 0, 0, r, rj, flat) / cnt;
        } else {
            const double* fd = a.aux_fine + a.fine_aux_stride + fsrc;   // depth plane
            double ws = 0.0;
            for (int p = 0; p < r; ++p)
                for (int q = 0; q < rj; ++q) ws = ws + (fd[(int64_t)p * fpitch + q] > 0.0 ? 1.0 : 0.0);
            const bool wetc = a.aux_coarse[a.coarse_aux_stride + cdst] > 0.0;
            if (!(ws > 0.0 && wetc)) continue;
#pragma unroll
            for (int c = 0; c < M; ++c)
                a.q_coarse[c * a.coarse_comp_stride + cdst] =
                    block_sum(a.q_fine + c * a.fine_comp_stride + fsrc, fd, fpitch, 0, 0, r, rj, flat) / ws;
        }
    }
}

// Planned restriction, 2D acoustics-type state (no wet weighting), fixed
// ratio R in both axes: every fine value of a coarse cell (all components)
// is loaded before the first store, so the loads of one cell form a single
// round trip (the generic loop above re-loads after each component's store,
// which the compiler must assume may alias).  Same summation order as
// block_sum (row sums, then their running total; the flat numpy order for a
// one-cell-wide overlap box goes through block_sum), so bitwise equal.
template <int M, int R>
__global__ void __launch_bounds__(256) k4_cells_r(AdjRestrictArgs a) {
    pdl_wait();
    pdl_trigger();
    const double cnt = (double)(R * R);
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.ncell) return;
    const int cdst = a.cell_dst[t], fsrc = a.cell_src[t], meta = a.cell_meta[t];
    const int fpitch = meta >> 1;
    double out[M];
    if (meta & 1) {
#pragma unroll
        for (int c = 0; c < M; ++c)
            out[c] = block_sum(a.q_fine + c * a.fine_comp_stride + fsrc, nullptr, fpitch, 0, 0, R, R, true) / cnt;
    } else {
        double v[M][R][R];
#pragma unroll
        for (int c = 0; c < M; ++c)
#pragma unroll
            for (int p = 0; p < R; ++p)
#pragma unroll
                for (int q = 0; q < R; ++q)
                    v[c][p][q] = __ldg(a.q_fine + c * a.fine_comp_stride + fsrc + (int64_t)p * fpitch + q);
#pragma unroll
        for (int c = 0; c < M; ++c) {
            double tot = 0.0;
#pragma unroll
            for (int p = 0; p < R; ++p) {
                double s = v[c][p][0];
#pragma unroll
                for (int q = 1; q < R; ++q) s = s + v[c][p][q];
                tot = p == 0 ? s : tot + s;
            }
            out[c] = tot / cnt;
        }
    }
#pragma unroll
    for (int c = 0; c < M; ++c) a.q_coarse[c * a.coarse_comp_stride + cdst] = out[c];
}

int restrict_level(const AdjRestrictArgs& a) {
    if (a.cell_dst) {
        if (a.ncell <= 0) return ADJ_OK;
        const cudaStream_t st = (cudaStream_t)a.stream;
        if (a.ndim == 2 && !a.swe && a.m == 3 && (a.ratio == 2 || a.ratio == 4)) {
            const dim3 g((a.ncell + 255) / 256), b(256);
            if (a.ratio == 2) launch_pdl(k4_cells_r<3, 2>, g, b, 0, st, a);
            else launch_pdl(k4_cells_r<3, 4>, g, b, 0, st, a);
            return check_launch("k4_cells_r");
        }
        int blocks = (a.ncell + 255) / 256;
        if (blocks > 148 * 8) blocks = 148 * 8;
        const dim3 g(blocks), b(256);
        if (a.m == 3 && !a.swe) launch_pdl(k4_cells<3, false>, g, b, 0, st, a);
        else if (a.m == 3) launch_pdl(k4_cells<3, true>, g, b, 0, st, a);
        else if (a.m == 2 && !a.swe) launch_pdl(k4_cells<2, false>, g, b, 0, st, a);
        else return ADJ_ERR_BAD_ARG;
        return check_launch("k4_cells");
    }
    if (a.nrect <= 0) return ADJ_OK;
    int threads = a.max_rect_cells >= 256 ? 256 : (a.max_rect_cells >= 128 ? 128 : 64);
    launch_pdl(k4_restrict, dim3(a.nrect), dim3(threads), 0, (cudaStream_t)a.stream, a);
    return check_launch("k4_restrict");
}

}  // namespace adj
