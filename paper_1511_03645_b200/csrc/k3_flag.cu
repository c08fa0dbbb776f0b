// K3: adjoint inner-product flagging with bit-packed output.  Compiled with
// -fmad=false so the inner products are bitwise identical to the reference:
//   inner_product_field / inner_product_flags   adjoint.py:227-257
//   interpolate_uniform / _axis_weights         geometry.py:248-290
//   _adjoint_dry_at                             adjoint.py:217-224
//   AdjointSnapshotStore.interpolate_time       adjoint.py:98-110  (mode 1)
//   evaluate_J / _uncovered_mask               adjoint.py:280-336  (k3_functional)
//   interpolate_patch (gauges)                  geometry.py:302-327 (k3_gauges)
//
// One thread per forward interior cell; a warp covers 32 consecutive cells of
// one patch (row-major over the interior), so the warp's ballot is exactly
// one 32-bit flag word and its popcount the raw flagged count.
#include "adj_common.cuh"
#include <stdlib.h>

namespace adj {

ADJ_D void uweights(double coord, double origin, double width, int n, int* i0, double* w) {
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

// Cells per thread: thread l of warp w handles cells base + 32 k + l, k < NC,
// so iteration k of a warp covers 32 consecutive cells = one flag word.
constexpr int NC = 4;

template <int M, bool TWO_D, bool TABLES>
__device__ __forceinline__ double cell_best(const AdjFlagArgs& a, const AdjPatch& p, int pidx, unsigned cidx,
                                            int64_t& o_out) {
    const int i = (int)(cidx / (unsigned)p.ny), j = (int)(cidx % (unsigned)p.ny);
    const int g = a.ghost;
    const int gy = TWO_D ? g : 0;
    const int64_t o = p.offset + (int64_t)(i + g) * p.pitch + (j + gy);
    o_out = o;
    double q[M];
#pragma unroll
    for (int c = 0; c < M; ++c) q[c] = a.q[c * a.comp_stride + o];
    int i0, j0 = 0, ia = 0, ja = 0;
    double wx, wy = 0.0;
    if (TABLES) {
        // host-precomputed per row / column (same arithmetic; bounds checked on the host)
        const int64_t ro = a.axis_off[2 * pidx] + i, co = a.axis_off[2 * pidx + 1] + j;
        i0 = a.axis_i[ro]; wx = a.axis_w[ro];
        if (TWO_D) { j0 = a.axis_i[co]; wy = a.axis_w[co]; }
        if (TWO_D && a.axis_dry) { ia = a.axis_dry[ro]; ja = a.axis_dry[co]; }
    } else {
        // cell centre (PatchSpec.cell_centers, geometry.py:67-74)
        const double x = a.origin_x + ((p.lo_x + i) + 0.5) * a.dx;
        const double y = TWO_D ? a.origin_y + ((p.lo_y + j) + 0.5) * a.dy : 0.0;
        // bounds check of interpolate_uniform (geometry.py:271-283); the
        // reference derives eps from the x extent and applies it to both axes
        const double hx = a.a_origin_x + a.nxa * a.a_dx;
        const double eps = 1e-12 * fmax(fabs(hx - a.a_origin_x), 1.0);
        bool oob = (x < a.a_origin_x - eps) || (x > hx + eps);
        if (TWO_D) {
            const double hy = a.a_origin_y + a.nya * a.a_dy;
            oob |= (y < a.a_origin_y - eps) || (y > hy + eps);
        }
        if (oob) atomicOr(a.status, 1);
        uweights(x, a.a_origin_x, a.a_dx, a.nxa, &i0, &wx);
        if (TWO_D) uweights(y, a.a_origin_y, a.a_dy, a.nya, &j0, &wy);
        if (TWO_D) {
            // _adjoint_dry_at: astype(int) truncates toward zero, then clip
            ia = (int)((x - a.a_origin_x) / a.a_dx);
            ja = (int)((y - a.a_origin_y) / a.a_dy);
            ia = ia < 0 ? 0 : (ia > a.nxa - 1 ? a.nxa - 1 : ia);
            ja = ja < 0 ? 0 : (ja > a.nya - 1 ? a.nya - 1 : ja);
        }
    }
    const int i1 = min(i0 + 1, a.nxa - 1);
    const int j1 = TWO_D ? min(j0 + 1, a.nya - 1) : 0;
    const unsigned plane = (unsigned)a.nxa * (unsigned)a.nya;
    const unsigned o00 = (unsigned)i0 * a.nya + j0, o10 = (unsigned)i1 * a.nya + j0;
    const unsigned o01 = (unsigned)i0 * a.nya + j1, o11 = (unsigned)i1 * a.nya + j1;
    const double ux = 1.0 - wx, uy = 1.0 - wy;
    double best = 0.0;
    for (int n = 0; n < a.nidx; ++n) {
        const int k = a.snap_index[n];
        double dot = 0.0;
        if (a.mode == 0 || k < 0) {
            const int kk = k < 0 ? -k - 1 : k;
            const double* f = a.ring + (int64_t)kk * plane * M;
#pragma unroll
            for (int c = 0; c < M; ++c) {
                const double* fc = f + c * plane;
                double qh;
                if (TWO_D)
                    qh = fc[o00] * ux * uy + fc[o10] * wx * uy + fc[o01] * ux * wy + fc[o11] * wx * wy;
                else
                    qh = fc[o00] * ux + fc[o10] * wx;
                dot = c == 0 ? qh * q[c] : dot + qh * q[c];
            }
        } else {
            // interpolate_time: vals = (1-w)*f[k] + w*f[k+1], then spatial interpolation
            const double w = a.interp_w[n];
            const double* fa = a.ring + (int64_t)k * plane * M;
            const double* fb = fa + (int64_t)plane * M;
#pragma unroll
            for (int c = 0; c < M; ++c) {
                const double* ac = fa + c * plane;
                const double* bc = fb + c * plane;
                double v00 = (1.0 - w) * ac[o00] + w * bc[o00];
                double v10 = (1.0 - w) * ac[o10] + w * bc[o10];
                double qh;
                if (TWO_D) {
                    double v01 = (1.0 - w) * ac[o01] + w * bc[o01];
                    double v11 = (1.0 - w) * ac[o11] + w * bc[o11];
                    qh = v00 * ux * uy + v10 * wx * uy + v01 * ux * wy + v11 * wx * wy;
                } else {
                    qh = v00 * ux + v10 * wx;
                }
                dot = c == 0 ? qh * q[c] : dot + qh * q[c];
            }
        }
        best = fmax(best, fabs(dot));
    }
    if (a.swe && !(a.aux[a.aux_stride + o] > 0.0)) best = 0.0;   // forward dry cell
    if (TWO_D && a.adj_wet != nullptr && !a.adj_wet[(unsigned)ia * a.nya + ja]) best = 0.0;
    return best;
}

template <int M, bool TWO_D, bool TABLES>
__global__ void __launch_bounds__(256) k3_flag(AdjFlagArgs a) {
    const int pidx = blockIdx.y;
    const AdjPatch p = a.patches[pidx];
    const unsigned ncell = (unsigned)p.nx * (unsigned)p.ny;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned base = (blockIdx.x * (blockDim.x >> 5) + warp) * (32u * NC);
    if (base >= ncell) return;
    unsigned long long cnt = 0;
#pragma unroll
    for (int kk = 0; kk < NC; ++kk) {
        const unsigned wbase = base + 32u * kk;
        if (wbase >= ncell) break;                     // warp-uniform
        const unsigned cidx = wbase + lane;
        bool flag = false;
        if (cidx < ncell) {
            int64_t o;
            const double best = cell_best<M, TWO_D, TABLES>(a, p, pidx, cidx, o);
            flag = best > a.tolerance;
            if (a.best != nullptr) a.best[a.best_offset[pidx] + cidx] = best;
        }
        const unsigned word = __ballot_sync(0xffffffffu, flag);
        if (lane == 0) a.flag_bits[p.flag_word + (wbase >> 5)] = word;
        cnt += __popc(word);
    }
    if (lane == 0 && cnt) atomicAdd(&a.counts[pidx], cnt);
}

// ---------------------------------------------------------------------------
// Table path, v2: the same per-cell arithmetic as cell_best<.., TABLES=true>
// (bitwise), restructured for issue efficiency -- mode as a template
// parameter, the window's snapshot list staged in shared memory, one
// division per thread (cells then advance by 32), per-snapshot component
// base pointers with 32-bit corner indices (one IMAD.WIDE per load).
constexpr int K3_MAXN = 256;

// 8-byte load at a 32-bit byte offset from a (warp-uniform) base
ADJ_D double ld(const char* base, unsigned off) { return *reinterpret_cast<const double*>(base + off); }

template <int M, bool TWO_D, bool MODE1>
__global__ void __launch_bounds__(256) k3_flag_t(AdjFlagArgs a) {
    __shared__ int s_k[K3_MAXN];
    __shared__ double s_w[K3_MAXN];
    const int nidx = a.nidx;
    for (int n = threadIdx.x; n < nidx; n += blockDim.x) {
        s_k[n] = a.snap_index[n];
        if (MODE1) s_w[n] = a.interp_w[n];
    }
    __syncthreads();
    const int pidx = blockIdx.y;
    const AdjPatch p = a.patches[pidx];
    const unsigned ny = TWO_D ? (unsigned)p.ny : 1u;
    const unsigned ncell = (unsigned)p.nx * ny;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned base = (blockIdx.x * (blockDim.x >> 5) + warp) * (32u * NC);
    if (base >= ncell) return;
    const int g = a.ghost, gy = TWO_D ? g : 0;
    const unsigned nxa = (unsigned)a.nxa, nya = (unsigned)a.nya;
    const int64_t plane_b = (int64_t)nxa * nya * 8;        // one snapshot component, bytes
    const int64_t snap_b = plane_b * M;                    // one snapshot, bytes
    const char* ring = reinterpret_cast<const char*>(a.ring);
    const int64_t rowoff = a.axis_off[2 * pidx], coloff = a.axis_off[2 * pidx + 1];
    unsigned i = TWO_D ? (base + lane) / ny : base + lane;
    unsigned j = TWO_D ? (base + lane) - i * ny : 0u;
    unsigned long long cnt = 0;
#pragma unroll
    for (int kk = 0; kk < NC; ++kk) {
        const unsigned wbase = base + 32u * kk;
        if (wbase >= ncell) break;                     // warp-uniform
        const unsigned cidx = wbase + lane;
        bool flag = false;
        if (cidx < ncell) {
            const int64_t o = p.offset + (int64_t)(i + g) * p.pitch + (j + gy);
            double q[M];
#pragma unroll
            for (int c = 0; c < M; ++c) q[c] = a.q[c * a.comp_stride + o];
            const int64_t ro = rowoff + i, co = coloff + j;
            const int i0 = a.axis_i[ro];
            const double wx = a.axis_w[ro];
            int j0 = 0;
            double wy = 0.0;
            if (TWO_D) { j0 = a.axis_i[co]; wy = a.axis_w[co]; }
            const unsigned i1 = min((unsigned)i0 + 1u, nxa - 1u);
            const unsigned j1 = TWO_D ? min((unsigned)j0 + 1u, nya - 1u) : 0u;
            // corner byte offsets within one snapshot component (plane * 8 < 2^32)
            const unsigned b00 = ((unsigned)i0 * nya + (unsigned)j0) * 8u, b10 = (i1 * nya + (unsigned)j0) * 8u;
            const unsigned b01 = ((unsigned)i0 * nya + j1) * 8u, b11 = (i1 * nya + j1) * 8u;
            const double ux = 1.0 - wx, uy = 1.0 - wy;
            double best = 0.0;
            for (int n = 0; n < nidx; ++n) {
                const int k = s_k[n];
                double dot = 0.0;
                if (!MODE1 || k < 0) {
                    const char* f = ring + (int64_t)(k < 0 ? -k - 1 : k) * snap_b;
#pragma unroll
                    for (int c = 0; c < M; ++c) {
                        const char* fc = f + c * plane_b;
                        double qh;
                        if (TWO_D)
                            qh = ld(fc, b00) * ux * uy + ld(fc, b10) * wx * uy + ld(fc, b01) * ux * wy +
                                 ld(fc, b11) * wx * wy;
                        else
                            qh = ld(fc, b00) * ux + ld(fc, b10) * wx;
                        dot = c == 0 ? qh * q[c] : dot + qh * q[c];
                    }
                } else {
                    const double w = s_w[n];
                    const char* fa = ring + (int64_t)k * snap_b;
#pragma unroll
                    for (int c = 0; c < M; ++c) {
                        const char* ac = fa + c * plane_b;
                        const char* bc = ac + snap_b;
                        const double v00 = (1.0 - w) * ld(ac, b00) + w * ld(bc, b00);
                        const double v10 = (1.0 - w) * ld(ac, b10) + w * ld(bc, b10);
                        double qh;
                        if (TWO_D) {
                            const double v01 = (1.0 - w) * ld(ac, b01) + w * ld(bc, b01);
                            const double v11 = (1.0 - w) * ld(ac, b11) + w * ld(bc, b11);
                            qh = v00 * ux * uy + v10 * wx * uy + v01 * ux * wy + v11 * wx * wy;
                        } else {
                            qh = v00 * ux + v10 * wx;
                        }
                        dot = c == 0 ? qh * q[c] : dot + qh * q[c];
                    }
                }
                best = fmax(best, fabs(dot));
            }
            if (a.swe && !(a.aux[a.aux_stride + o] > 0.0)) best = 0.0;   // forward dry cell
            if (TWO_D && a.adj_wet != nullptr && a.axis_dry) {
                const int ia = a.axis_dry[ro], ja = a.axis_dry[co];
                if (!a.adj_wet[(unsigned)ia * nya + ja]) best = 0.0;
            }
            flag = best > a.tolerance;
            if (a.best != nullptr) a.best[a.best_offset[pidx] + cidx] = best;
        }
        const unsigned word = __ballot_sync(0xffffffffu, flag);
        if (lane == 0) a.flag_bits[p.flag_word + (wbase >> 5)] = word;
        cnt += __popc(word);
        // next cell of this lane: 32 further in row-major order
        if (TWO_D) { j += 32u; while (j >= ny) { j -= ny; ++i; } } else { i += 32u; }
    }
    if (lane == 0 && cnt) atomicAdd(&a.counts[pidx], cnt);
}

// ---------------------------------------------------------------------------
// Row layout (patch rows a multiple of 32*NC cells, e.g. C3/C4 and any patch
// of >=128-cell rows): a warp's 32*NC cells lie in one row i, so the row
// weights are warp-uniform and each component's two adjoint rows are uniform
// pointers; lane l's cells are columns j+32kk, whose state and column-table
// entries sit at immediate offsets.  Every load is issued before the first
// store.  Same per-cell arithmetic as k3_flag_t (bitwise); the adjoint axis
// tables never give a corner past the last row/column when nxa, nya >= 2
// (uweights clamps i0 <= n-2), which the host checks before choosing it.
#ifndef K3_ROW_PIPE
#define K3_ROW_PIPE 1
#endif
#ifndef K3_ROW_UNROLL
#define K3_ROW_UNROLL 0   // 0: the compiler's choice
#endif
#ifndef K3_ROW_NC
#define K3_ROW_NC 4
#endif
constexpr int K3_ROW_UNR = K3_ROW_UNROLL > 0 ? K3_ROW_UNROLL : 1;
constexpr int RNC = K3_ROW_NC;     // cells per lane (a warp's segment is 32*RNC columns)
constexpr int K3_ROW_WARPS = 4;   // warps per CTA
#ifndef K3_ROW_RUN_ROWS
#define K3_ROW_RUN_ROWS 0
#endif
constexpr int K3_ROW_RUN = K3_ROW_RUN_ROWS;   // rows one warp marches down (0: sized at launch to one wave)
#ifndef K3_ROW_DEPTH
#define K3_ROW_DEPTH 2
#endif
constexpr int RDEPTH = K3_ROW_DEPTH;          // state rows in flight per warp (shared-memory buffers)

template <bool MODE1>
#ifndef K3_ROW_MINB
#define K3_ROW_MINB 1
#endif
__global__ void __launch_bounds__(32 * K3_ROW_WARPS, K3_ROW_MINB) k3_row(AdjFlagArgs a, int run) {
    // warp = one 32*RNC-column segment of K3_ROW_RUN consecutive rows.  The
    // column tables load once; the next row's state streams into shared
    // memory (cp.async) and its row-table entry into registers while this
    // row is computed, so the corner loads depend on registers only, and
    // rows sharing adjoint rows (refinement ratio >= 2) hit L1.
    __shared__ double s_q[K3_ROW_WARPS][RDEPTH][RNC * 3][32];
    const int pidx = blockIdx.z;
    const AdjPatch p = a.patches[pidx];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned seg = blockIdx.y * K3_ROW_WARPS + warp;          // column segment
    const unsigned nseg = (unsigned)p.ny / (32u * RNC);
    const unsigned r0 = blockIdx.x * (unsigned)run;
    if (seg >= nseg || r0 >= (unsigned)p.nx) return;               // warp-uniform
    const unsigned r1 = min(r0 + (unsigned)run, (unsigned)p.nx);
    const unsigned ny = (unsigned)p.ny, j = seg * (32u * RNC) + lane;
    const int g = a.ghost;
    const int64_t cs = a.comp_stride;
    const int64_t nya = a.nya;
    const int64_t plane = (int64_t)a.nxa * nya;
    const int k = __ldg(a.snap_index);
    const bool interp = MODE1 && k >= 0;
    const double* fa = a.ring + (int64_t)(k < 0 ? -k - 1 : k) * plane * 3;
    const double w = interp ? __ldg(a.interp_w) : 0.0;
    const int64_t rowoff = a.axis_off[2 * pidx], coloff = a.axis_off[2 * pidx + 1];
    const double* qcol = a.q + p.offset + (int64_t)g * p.pitch + g + j;

    auto prefetch = [&](unsigned i, int buf) {
        const double* qp = qcol + (int64_t)i * p.pitch;
#pragma unroll
        for (int kk = 0; kk < RNC; ++kk)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const unsigned dst = (unsigned)__cvta_generic_to_shared(&s_q[warp][buf][kk * 3 + cc][lane]);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(qp + cc * cs + 32 * kk)
                             : "memory");
            }
    };
#pragma unroll
    for (int d = 0; d < RDEPTH - 1; ++d) {       // rows r0 .. r0+RDEPTH-2 in flight
        if (r0 + d < r1) prefetch(r0 + d, d);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }

    double wy[RNC], uy[RNC];
    int j0[RNC], ja[RNC];
#pragma unroll
    for (int kk = 0; kk < RNC; ++kk) {
        j0[kk] = __ldg(a.axis_i + coloff + j + 32 * kk);
        wy[kk] = __ldg(a.axis_w + coloff + j + 32 * kk);
        uy[kk] = 1.0 - wy[kk];
        ja[kk] = a.axis_dry ? __ldg(a.axis_dry + coloff + j + 32 * kk) : 0;
    }
    auto row_epilogue = [&](unsigned i, double (&best)[RNC], unsigned long long& cnt) {
        if (a.swe) {   // forward dry cells
            const double* cp = a.aux + a.aux_stride + p.offset + (int64_t)(i + g) * p.pitch + (j + g);
#pragma unroll
            for (int kk = 0; kk < RNC; ++kk)
                if (!(__ldg(cp + 32 * kk) > 0.0)) best[kk] = 0.0;
        }
        if (a.adj_wet != nullptr && a.axis_dry) {   // adjoint cell containing the centre is dry
            const int ia = __ldg(a.axis_dry + rowoff + i);
#pragma unroll
            for (int kk = 0; kk < RNC; ++kk)
                if (!a.adj_wet[(int64_t)ia * nya + ja[kk]]) best[kk] = 0.0;
        }
        const unsigned base = i * ny + seg * (32u * RNC);
#pragma unroll
        for (int kk = 0; kk < RNC; ++kk) {
            if (a.best != nullptr) a.best[a.best_offset[pidx] + base + 32u * kk + lane] = best[kk];
            const unsigned word = __ballot_sync(0xffffffffu, best[kk] > a.tolerance);
            if (lane == 0) a.flag_bits[p.flag_word + ((base >> 5) + kk)] = word;
            cnt += __popc(word);
        }
    };
    int i0 = __ldg(a.axis_i + rowoff + r0);
    double wx = __ldg(a.axis_w + rowoff + r0);
    unsigned long long cnt = 0;
    int buf = 0;
#if K3_ROW_PIPE
    if (!MODE1) {
        // mode 0: the next row's corners load into registers as soon as this
        // row's interpolation has consumed them, so they fly during the dot
        // products, ballots and stores
        double C[RNC][3][4];
        auto corners = [&](int ii0) {
#pragma unroll
            for (int kk = 0; kk < RNC; ++kk)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double* q0 = fa + c * plane + (int64_t)ii0 * nya + j0[kk];
                    C[kk][c][0] = __ldg(q0); C[kk][c][1] = __ldg(q0 + nya);
                    C[kk][c][2] = __ldg(q0 + 1); C[kk][c][3] = __ldg(q0 + nya + 1);
                }
        };
        corners(i0);
        int i0n = r0 + 1 < r1 ? __ldg(a.axis_i + rowoff + r0 + 1) : 0;
        double wxn = r0 + 1 < r1 ? __ldg(a.axis_w + rowoff + r0 + 1) : 0.0;
#if K3_ROW_UNROLL > 0
#pragma unroll K3_ROW_UNR
#endif
        for (unsigned i = r0; i < r1; ++i, buf = buf + 1 == RDEPTH ? 0 : buf + 1) {
            const bool more = i + 1 < r1;
            if (i + RDEPTH - 1 < r1) prefetch(i + RDEPTH - 1, buf == 0 ? RDEPTH - 1 : buf - 1);
            asm volatile("cp.async.commit_group;\n" ::: "memory");
            const double ux = 1.0 - wx;
            double qh[RNC][3];
#pragma unroll
            for (int kk = 0; kk < RNC; ++kk)
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    qh[kk][c] = C[kk][c][0] * ux * uy[kk] + C[kk][c][1] * wx * uy[kk] + C[kk][c][2] * ux * wy[kk] +
                                C[kk][c][3] * wx * wy[kk];
            if (more) corners(i0n);
            const bool more2 = i + 2 < r1;
            const int i0nn = more2 ? __ldg(a.axis_i + rowoff + i + 2) : 0;
            const double wxnn = more2 ? __ldg(a.axis_w + rowoff + i + 2) : 0.0;
            asm volatile("cp.async.wait_group %0;\n" ::"n"(RDEPTH - 1) : "memory");
            __syncwarp();
            double best[RNC];
#pragma unroll
            for (int kk = 0; kk < RNC; ++kk) {
                double dot = 0.0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double qc = s_q[warp][buf][kk * 3 + c][lane];
                    dot = c == 0 ? qh[kk][c] * qc : dot + qh[kk][c] * qc;
                }
                best[kk] = fmax(0.0, fabs(dot));
            }
            __syncwarp();
            row_epilogue(i, best, cnt);
            wx = wxn; wxn = wxnn; i0n = i0nn;
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        if (lane == 0 && cnt) atomicAdd(&a.counts[pidx], cnt);
        return;
    }
#endif
    for (unsigned i = r0; i < r1; ++i, buf = buf + 1 == RDEPTH ? 0 : buf + 1) {
        const bool more = i + 1 < r1;
        if (i + RDEPTH - 1 < r1) prefetch(i + RDEPTH - 1, buf == 0 ? RDEPTH - 1 : buf - 1);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        const int i0n = more ? __ldg(a.axis_i + rowoff + i + 1) : 0;
        const double wxn = more ? __ldg(a.axis_w + rowoff + i + 1) : 0.0;

        const double ux = 1.0 - wx;
        double qh[RNC][3];
#pragma unroll
        for (int kk = 0; kk < RNC; ++kk) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double* q0 = fa + c * plane + (int64_t)i0 * nya + j0[kk];
                const double* q1 = q0 + nya;
                if (!interp) {
                    qh[kk][c] = __ldg(q0) * ux * uy[kk] + __ldg(q1) * wx * uy[kk] + __ldg(q0 + 1) * ux * wy[kk] +
                                __ldg(q1 + 1) * wx * wy[kk];
                } else {   // interpolate_time, then the spatial stencil (k3_flag_t's order)
                    const int64_t sb = plane * 3;
                    const double v00 = (1.0 - w) * __ldg(q0) + w * __ldg(q0 + sb);
                    const double v10 = (1.0 - w) * __ldg(q1) + w * __ldg(q1 + sb);
                    const double v01 = (1.0 - w) * __ldg(q0 + 1) + w * __ldg(q0 + 1 + sb);
                    const double v11 = (1.0 - w) * __ldg(q1 + 1) + w * __ldg(q1 + 1 + sb);
                    qh[kk][c] = v00 * ux * uy[kk] + v10 * wx * uy[kk] + v01 * ux * wy[kk] + v11 * wx * wy[kk];
                }
            }
        }
        asm volatile("cp.async.wait_group %0;\n" ::"n"(RDEPTH - 1) : "memory");   // this row's state has landed
        __syncwarp();
        double best[RNC];
#pragma unroll
        for (int kk = 0; kk < RNC; ++kk) {
            double dot = 0.0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double qc = s_q[warp][buf][kk * 3 + c][lane];
                dot = c == 0 ? qh[kk][c] * qc : dot + qh[kk][c] * qc;
            }
            best[kk] = fmax(0.0, fabs(dot));
        }
        __syncwarp();                                          // buffer free for the row after next
        row_epilogue(i, best, cnt);
        i0 = i0n;
        wx = wxn;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    if (lane == 0 && cnt) atomicAdd(&a.counts[pidx], cnt);
}

// ---------------------------------------------------------------------------
// 2D table path with two horizontally adjacent cells per lane: a warp covers
// 64 consecutive cells (two flag words).  When every lane's pair lies in one
// row with a common adjoint stencil (same j0 -- e.g. refinement ratio 4 on
// aligned pairs), each snapshot's 12 corner loads serve both cells; each
// cell's arithmetic is unchanged (bitwise).  Ballots of the even and odd
// cells are interleaved back into the standard word layout.
constexpr int NP = 2;   // pairs per lane

ADJ_D unsigned spread16(unsigned x) {   // bit k -> bit 2k
    x &= 0xffffu;
    x = (x | (x << 8)) & 0x00ff00ffu;
    x = (x | (x << 4)) & 0x0f0f0f0fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

// ---------------------------------------------------------------------------
// Row layout with column pairs (ADJ_FLAG_PAIRS; single-snapshot windows, mode
// 0): lane l owns the cell pairs (64pp + 2l, 64pp + 2l + 1), pp = 0, 1, of its
// warp's 128-column segment.  Both cells of a pair share the adjoint stencil
// column, so a row needs 12 corner loads per pair instead of 12 per cell, the
// corners prefetched a row ahead take half the registers, and the state row
// streams in as 16-byte cp.async pieces read back with one LDS.128.  Each
// cell's arithmetic is k3_row's (bitwise); the even/odd ballots are
// interleaved into the standard flag words.
#ifndef K3_ROWP_DEPTH
#define K3_ROWP_DEPTH 3   // state rows in flight per warp of k3_rowp (round 2: 3 measured 0.090 vs 0.094 ms
                          // with 2 on C4; 4 exceeds the static shared-memory limit)
#endif
constexpr int RPDEPTH = K3_ROWP_DEPTH;
#ifndef K3_ROWP_MINB
#define K3_ROWP_MINB 3
#endif
constexpr int NPR = 2;   // pairs per lane

__global__ void __launch_bounds__(32 * K3_ROW_WARPS, K3_ROWP_MINB) k3_rowp(AdjFlagArgs a, int run) {
    __shared__ double2 s_q[K3_ROW_WARPS][RPDEPTH][NPR * 3][32];
    const int pidx = blockIdx.z;
    const AdjPatch p = a.patches[pidx];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned seg = blockIdx.y * K3_ROW_WARPS + warp;
    const unsigned nseg = (unsigned)p.ny / 128u;
    const unsigned r0 = blockIdx.x * (unsigned)run;
    if (seg >= nseg || r0 >= (unsigned)p.nx) return;               // warp-uniform
    const unsigned r1 = min(r0 + (unsigned)run, (unsigned)p.nx);
    const unsigned ny = (unsigned)p.ny, j = seg * 128u + 2u * lane;   // pair pp: columns j + 64pp, +1
    const int g = a.ghost;
    const int64_t cs = a.comp_stride;
    const int64_t nya = a.nya;
    const int64_t plane = (int64_t)a.nxa * nya;
    const int k = __ldg(a.snap_index);
    const double* fa = a.ring + (int64_t)k * plane * 3;
    const int64_t rowoff = a.axis_off[2 * pidx], coloff = a.axis_off[2 * pidx + 1];
    const double* qcol = a.q + p.offset + (int64_t)g * p.pitch + g + j;   // 16-byte aligned (even column)

    auto prefetch = [&](unsigned i, int buf) {
        const double* qp = qcol + (int64_t)i * p.pitch;
#pragma unroll
        for (int pp = 0; pp < NPR; ++pp)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const unsigned dst = (unsigned)__cvta_generic_to_shared(&s_q[warp][buf][pp * 3 + cc][lane]);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(qp + cc * cs + 64 * pp)
                             : "memory");
            }
    };
#pragma unroll
    for (int d = 0; d < RPDEPTH - 1; ++d) {
        if (r0 + d < r1) prefetch(r0 + d, d);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    double wy[NPR][2], uy[NPR][2];
    int ja[NPR][2];
    unsigned off[NPR][3];
    const char* fab = reinterpret_cast<const char*>(fa);
    const int64_t rowbytes = nya * 8;
#pragma unroll
    for (int pp = 0; pp < NPR; ++pp) {
        const int jt = (int)(j + 64 * pp);
        const int j0 = __ldg(a.axis_i + coloff + jt);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            wy[pp][e] = __ldg(a.axis_w + coloff + jt + e);
            uy[pp][e] = 1.0 - wy[pp][e];
            ja[pp][e] = a.axis_dry ? __ldg(a.axis_dry + coloff + jt + e) : 0;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) off[pp][c] = (unsigned)(((int64_t)c * plane + j0) * 8);
    }
    double C[NPR][3][4];
    auto corners = [&](int ii0) {
        const char* b0 = fab + ii0 * rowbytes;
        const char* b1 = b0 + rowbytes;
#pragma unroll
        for (int pp = 0; pp < NPR; ++pp)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double* q0 = reinterpret_cast<const double*>(b0 + off[pp][c]);
                const double* q1 = reinterpret_cast<const double*>(b1 + off[pp][c]);
                C[pp][c][0] = __ldg(q0); C[pp][c][1] = __ldg(q1);
                C[pp][c][2] = __ldg(q0 + 1); C[pp][c][3] = __ldg(q1 + 1);
            }
    };
    double wx = __ldg(a.axis_w + rowoff + r0);
    corners(__ldg(a.axis_i + rowoff + r0));
    int i0n = r0 + 1 < r1 ? __ldg(a.axis_i + rowoff + r0 + 1) : 0;
    double wxn = r0 + 1 < r1 ? __ldg(a.axis_w + rowoff + r0 + 1) : 0.0;
    unsigned long long cnt = 0;
    int buf = 0;
    for (unsigned i = r0; i < r1; ++i, buf = buf + 1 == RPDEPTH ? 0 : buf + 1) {
        const bool more = i + 1 < r1;
        if (i + RPDEPTH - 1 < r1) prefetch(i + RPDEPTH - 1, buf == 0 ? RPDEPTH - 1 : buf - 1);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        const double ux = 1.0 - wx;
        double qh[NPR][2][3];
#pragma unroll
        for (int pp = 0; pp < NPR; ++pp)
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    qh[pp][e][c] = C[pp][c][0] * ux * uy[pp][e] + C[pp][c][1] * wx * uy[pp][e] +
                                   C[pp][c][2] * ux * wy[pp][e] + C[pp][c][3] * wx * wy[pp][e];
        if (more) corners(i0n);
        const bool more2 = i + 2 < r1;
        const int i0nn = more2 ? __ldg(a.axis_i + rowoff + i + 2) : 0;
        const double wxnn = more2 ? __ldg(a.axis_w + rowoff + i + 2) : 0.0;
        asm volatile("cp.async.wait_group %0;\n" ::"n"(RPDEPTH - 1) : "memory");
        __syncwarp();
        double best[NPR][2];
#pragma unroll
        for (int pp = 0; pp < NPR; ++pp) {
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double2 qc = s_q[warp][buf][pp * 3 + c][lane];
                d0 = c == 0 ? qh[pp][0][c] * qc.x : d0 + qh[pp][0][c] * qc.x;
                d1 = c == 0 ? qh[pp][1][c] * qc.y : d1 + qh[pp][1][c] * qc.y;
            }
            best[pp][0] = fmax(0.0, fabs(d0));
            best[pp][1] = fmax(0.0, fabs(d1));
        }
        __syncwarp();
        if (a.swe) {   // forward dry cells
            const double* cp = a.aux + a.aux_stride + p.offset + (int64_t)(i + g) * p.pitch + (j + g);
#pragma unroll
            for (int pp = 0; pp < NPR; ++pp)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (!(__ldg(cp + 64 * pp + e) > 0.0)) best[pp][e] = 0.0;
        }
        if (a.adj_wet != nullptr && a.axis_dry) {   // adjoint cell containing the centre is dry
            const int ia = __ldg(a.axis_dry + rowoff + i);
#pragma unroll
            for (int pp = 0; pp < NPR; ++pp)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (!a.adj_wet[(int64_t)ia * nya + ja[pp][e]]) best[pp][e] = 0.0;
        }
        const unsigned base = i * ny + seg * 128u;
        if (a.best != nullptr) {
#pragma unroll
            for (int pp = 0; pp < NPR; ++pp)
                *reinterpret_cast<double2*>(a.best + a.best_offset[pidx] + base + 64u * pp + 2u * lane) =
                    make_double2(best[pp][0], best[pp][1]);
        }
        // flag words: word 2pp+h, bit b is cell 64pp + 32h + b, held by lane
        // 16h + b/2 as its pair element b%2.  Each lane fetches the 4 flag bits
        // of lanes l/2 and 16 + l/2 and the four ballots are the words.
        unsigned bits = 0;
#pragma unroll
        for (int pp = 0; pp < NPR; ++pp)
            bits |= (best[pp][0] > a.tolerance ? 1u : 0u) << (2 * pp) | (best[pp][1] > a.tolerance ? 2u : 0u) << (2 * pp);
        const unsigned t0 = __shfl_sync(0xffffffffu, bits, lane >> 1) >> (lane & 1);
        const unsigned t1 = __shfl_sync(0xffffffffu, bits, 16 + (lane >> 1)) >> (lane & 1);
        unsigned words[4];
#pragma unroll
        for (int pp = 0; pp < NPR; ++pp) {
            words[2 * pp] = __ballot_sync(0xffffffffu, (t0 >> (2 * pp)) & 1u);
            words[2 * pp + 1] = __ballot_sync(0xffffffffu, (t1 >> (2 * pp)) & 1u);
        }
        if (lane < 4) {
            const unsigned wv = lane == 0 ? words[0] : (lane == 1 ? words[1] : (lane == 2 ? words[2] : words[3]));
            a.flag_bits[p.flag_word + (base >> 5) + lane] = wv;
        }
        cnt += __popc(words[0]) + __popc(words[1]) + __popc(words[2]) + __popc(words[3]);
        wx = wxn; wxn = wxnn; i0n = i0nn;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    if (lane == 0 && cnt) atomicAdd(&a.counts[pidx], cnt);
}


// qhat from the four corners: the reference's order (EXACT, bitwise) or, FAST,
// per-cell corner weights W = (ux uy, wx uy, ux wy, wx wy) and FMAs
template <bool FASTW>
ADJ_D double corner_interp(double v00, double v10, double v01, double v11, double ux, double uy, double wx,
                           double wy, const double (&W)[4]) {
    if (FASTW) return fma(v11, W[3], fma(v01, W[2], fma(v10, W[1], v00 * W[0])));
    return v00 * ux * uy + v10 * wx * uy + v01 * ux * wy + v11 * wx * wy;
}

template <bool MODE1, bool SHARED, bool FASTW>
ADJ_D void pair_window(const AdjFlagArgs& a, const int* s_k, const double* s_w, int nidx, const char* ring,
                       int64_t plane_b, int64_t snap_b, const double (&q)[2][3], const unsigned (&b)[2][4],
                       const double (&ux)[2], const double (&uy)[2], const double (&wx)[2], const double (&wy)[2],
                       double (&best)[2]) {
    double W[2][4];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        W[e][0] = ux[e] * uy[e]; W[e][1] = wx[e] * uy[e]; W[e][2] = ux[e] * wy[e]; W[e][3] = wx[e] * wy[e];
    }
    for (int n = 0; n < nidx; ++n) {
        const int k = s_k[n];
        double dot[2] = {0.0, 0.0};
        if (!MODE1 || k < 0) {
            const char* f = ring + (int64_t)(k < 0 ? -k - 1 : k) * snap_b;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const char* fc = f + c * plane_b;
                const double v00 = ld(fc, b[0][0]), v10 = ld(fc, b[0][1]), v01 = ld(fc, b[0][2]), v11 = ld(fc, b[0][3]);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    double w00 = v00, w10 = v10, w01 = v01, w11 = v11;
                    if (!SHARED && e == 1) {
                        w00 = ld(fc, b[1][0]); w10 = ld(fc, b[1][1]); w01 = ld(fc, b[1][2]); w11 = ld(fc, b[1][3]);
                    }
                    const double qh = corner_interp<FASTW>(w00, w10, w01, w11, ux[e], uy[e], wx[e], wy[e], W[e]);
                    dot[e] = c == 0 ? qh * q[e][c] : (FASTW ? fma(qh, q[e][c], dot[e]) : dot[e] + qh * q[e][c]);
                }
            }
        } else {   // interpolate_time, then the spatial stencil
            const double w = s_w[n];
            const char* fa = ring + (int64_t)k * snap_b;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const char* ac = fa + c * plane_b;
                const char* bc = ac + snap_b;
                double t00 = (1.0 - w) * ld(ac, b[0][0]) + w * ld(bc, b[0][0]);
                double t10 = (1.0 - w) * ld(ac, b[0][1]) + w * ld(bc, b[0][1]);
                double t01 = (1.0 - w) * ld(ac, b[0][2]) + w * ld(bc, b[0][2]);
                double t11 = (1.0 - w) * ld(ac, b[0][3]) + w * ld(bc, b[0][3]);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    if (!SHARED && e == 1) {
                        t00 = (1.0 - w) * ld(ac, b[1][0]) + w * ld(bc, b[1][0]);
                        t10 = (1.0 - w) * ld(ac, b[1][1]) + w * ld(bc, b[1][1]);
                        t01 = (1.0 - w) * ld(ac, b[1][2]) + w * ld(bc, b[1][2]);
                        t11 = (1.0 - w) * ld(ac, b[1][3]) + w * ld(bc, b[1][3]);
                    }
                    const double qh = corner_interp<FASTW>(t00, t10, t01, t11, ux[e], uy[e], wx[e], wy[e], W[e]);
                    dot[e] = c == 0 ? qh * q[e][c] : (FASTW ? fma(qh, q[e][c], dot[e]) : dot[e] + qh * q[e][c]);
                }
            }
        }
        best[0] = fmax(best[0], fabs(dot[0]));
        best[1] = fmax(best[1], fabs(dot[1]));
    }
}

template <bool MODE1, bool FASTW>
__global__ void __launch_bounds__(256, 3) k3_pair(AdjFlagArgs a) {
    __shared__ int s_k[K3_MAXN];
    __shared__ double s_w[K3_MAXN];
    const int nidx = a.nidx;
    for (int n = threadIdx.x; n < nidx; n += blockDim.x) {
        s_k[n] = a.snap_index[n];
        if (MODE1) s_w[n] = a.interp_w[n];
    }
    __syncthreads();
    const int pidx = blockIdx.y;
    const AdjPatch p = a.patches[pidx];
    const unsigned ny = (unsigned)p.ny;
    const unsigned ncell = (unsigned)p.nx * ny;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned base = (blockIdx.x * (blockDim.x >> 5) + warp) * (64u * NP);
    if (base >= ncell) return;
    const int g = a.ghost;
    const unsigned nxa = (unsigned)a.nxa, nya = (unsigned)a.nya;
    const int64_t plane_b = (int64_t)nxa * nya * 8;
    const int64_t snap_b = plane_b * 3;
    const char* ring = reinterpret_cast<const char*>(a.ring);
    const int64_t rowoff = a.axis_off[2 * pidx], coloff = a.axis_off[2 * pidx + 1];
    unsigned i = (base + 2u * lane) / ny;
    unsigned j = (base + 2u * lane) - i * ny;
    unsigned long long cnt = 0;
#pragma unroll
    for (int kk = 0; kk < NP; ++kk) {
        const unsigned wbase = base + 64u * kk;
        if (wbase >= ncell) break;                     // warp-uniform
        const unsigned ca = wbase + 2u * lane;
        bool live[2] = {ca < ncell, ca + 1u < ncell};
        const bool same_row = j + 1u < ny;
        const unsigned ci[2] = {i, same_row ? i : i + 1u}, cj[2] = {j, same_row ? j + 1u : 0u};
        double q[2][3], ux[2], uy[2], wx[2], wy[2], best[2] = {0.0, 0.0};
        unsigned b[2][4];
        int j0s[2] = {0, 0}, i0s[2] = {0, 0};
        int64_t o[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const unsigned ii = live[e] ? ci[e] : 0u, jj = live[e] ? cj[e] : 0u;
            o[e] = p.offset + (int64_t)(ii + g) * p.pitch + (jj + g);
#pragma unroll
            for (int c = 0; c < 3; ++c) q[e][c] = live[e] ? a.q[c * a.comp_stride + o[e]] : 0.0;
            const int i0 = live[e] ? a.axis_i[rowoff + ii] : 0;
            const int j0 = live[e] ? a.axis_i[coloff + jj] : 0;
            wx[e] = live[e] ? a.axis_w[rowoff + ii] : 0.0;
            wy[e] = live[e] ? a.axis_w[coloff + jj] : 0.0;
            const unsigned i1 = min((unsigned)i0 + 1u, nxa - 1u), j1 = min((unsigned)j0 + 1u, nya - 1u);
            b[e][0] = ((unsigned)i0 * nya + (unsigned)j0) * 8u;
            b[e][1] = (i1 * nya + (unsigned)j0) * 8u;
            b[e][2] = ((unsigned)i0 * nya + j1) * 8u;
            b[e][3] = (i1 * nya + j1) * 8u;
            ux[e] = 1.0 - wx[e];
            uy[e] = 1.0 - wy[e];
            i0s[e] = i0; j0s[e] = j0;
        }
        // one stencil for both cells of every lane -> shared corner loads
        const bool share = !live[1] || (same_row && i0s[0] == i0s[1] && j0s[0] == j0s[1]);
        if (__all_sync(0xffffffffu, share))
            pair_window<MODE1, true, FASTW>(a, s_k, s_w, nidx, ring, plane_b, snap_b, q, b, ux, uy, wx, wy, best);
        else
            pair_window<MODE1, false, FASTW>(a, s_k, s_w, nidx, ring, plane_b, snap_b, q, b, ux, uy, wx, wy, best);
        bool flag[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double bst = best[e];
            if (live[e]) {
                if (a.swe && !(a.aux[a.aux_stride + o[e]] > 0.0)) bst = 0.0;   // forward dry cell
                if (a.adj_wet != nullptr && a.axis_dry) {
                    const int ia = a.axis_dry[rowoff + ci[e]], ja = a.axis_dry[coloff + cj[e]];
                    if (!a.adj_wet[(unsigned)ia * nya + ja]) bst = 0.0;
                }
                if (a.best != nullptr) a.best[a.best_offset[pidx] + ca + e] = bst;
            }
            flag[e] = live[e] && bst > a.tolerance;
        }
        const unsigned be = __ballot_sync(0xffffffffu, flag[0]), bo = __ballot_sync(0xffffffffu, flag[1]);
        if (lane == 0) {
            const unsigned w0 = spread16(be) | (spread16(bo) << 1);
            const unsigned w1 = spread16(be >> 16) | (spread16(bo >> 16) << 1);
            a.flag_bits[p.flag_word + (wbase >> 5)] = w0;
            if (wbase + 32u < ncell) a.flag_bits[p.flag_word + (wbase >> 5) + 1] = w1;
            cnt += __popc(w0) + __popc(w1);
        }
        j += 64u;
        while (j >= ny) { j -= ny; ++i; }
    }
    if (lane == 0 && cnt) atomicAdd(&a.counts[pidx], cnt);
}

// ---------------------------------------------------------------------------
// Window envelope (AdjFlagArgs.envelope): env[c][node] = max over the window's
// snapshots of |ring[k][c][node]| (NaN propagates, so a non-finite field is
// never pruned).  Mode 1 entries cover both snapshots of their blend.
__global__ void k3_envelope(AdjFlagArgs a) {
    const int64_t plane = (int64_t)a.nxa * a.nya, snap = 3 * plane;
    const int nidx = a.nidx;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < plane; v += (int64_t)gridDim.x * blockDim.x) {
        double m0 = 0.0, m1 = 0.0, m2 = 0.0;
        auto take = [&](int k) {
            const double* f = a.ring + (int64_t)k * snap + v;
            const double x0 = fabs(__ldcs(f)), x1 = fabs(__ldcs(f + plane)), x2 = fabs(__ldcs(f + 2 * plane));
            m0 = (x0 > m0 || x0 != x0) ? x0 : m0;
            m1 = (x1 > m1 || x1 != x1) ? x1 : m1;
            m2 = (x2 > m2 || x2 != x2) ? x2 : m2;
        };
        for (int n = 0; n < nidx; ++n) {
            const int k = __ldg(a.snap_index + n);
            if (a.mode == 1 && k >= 0) { take(k); take(k + 1); }
            else take(k >= 0 ? k : -k - 1);
        }
        a.envelope[v] = m0;                  // node envelope, planes 0..2
        a.envelope[plane + v] = m1;
        a.envelope[2 * plane + v] = m2;
    }
}

ADJ_D double nanmax(double x, double m) { return (x > m || x != x) ? x : m; }


// ---------------------------------------------------------------------------
// Windows of >= 2 snapshots on the row layout with quads (ADJ_FLAG_QUADS:
// even-aligned row pairs and column pairs share their adjoint stencil, e.g.
// ratio 4 on aligned grids, C4).  Lane l owns the 2x2 cells (rows i, i+1;
// columns 64 seg + 2l, +1): one snapshot's 12 corner loads serve 4 cells, the
// next snapshot's corners load while this one is interpolated, the window
// list sits in shared memory and the warp marches down row pairs with the
// state streamed by cp.async.  EXACT: k3_row's per-cell arithmetic (bitwise);
// FAST: per-cell corner weights and FMAs.
#ifndef K3_QUAD_MINB
#define K3_QUAD_MINB 3       // EXACT: 168 registers (a few spilled bytes), 3 CTAs/SM
#endif
#ifndef K3_QUAD_MINB_FAST
#define K3_QUAD_MINB_FAST 2  // FAST: the corner weights need ~225 registers
#endif

#ifndef K3_QUAD_DEPTH
#define K3_QUAD_DEPTH 3   // snapshots of corners in registers (2: one ahead, 3: two ahead)
#endif

template <bool FASTW>
ADJ_D void quad_rows(const AdjFlagArgs& a, const char* const* s_base, double2 (*s_qw)[6][32], int pidx,
                     unsigned seg, unsigned r0, unsigned rend, int lane) {
    const int nidx = a.nidx;
    const AdjPatch p = a.patches[pidx];
    const unsigned nseg = (unsigned)p.ny / 64u;
    if (seg >= nseg || r0 >= (unsigned)p.nx) return;               // warp-uniform; no barrier below
    const unsigned r1 = min(rend, (unsigned)p.nx);                 // nx is even
    const unsigned ny = (unsigned)p.ny, j = seg * 64u + 2u * lane;
    const int g = a.ghost;
    const int64_t cs = a.comp_stride;
    const int64_t nya = a.nya;
    const int64_t plane = (int64_t)a.nxa * nya;
    const int64_t rowoff = a.axis_off[2 * pidx], coloff = a.axis_off[2 * pidx + 1];
    const double* qcol = a.q + p.offset + (int64_t)g * p.pitch + g + j;   // 16-byte aligned (even column)

    auto prefetch = [&](unsigned i, int buf) {   // rows i, i+1
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const unsigned dst = (unsigned)__cvta_generic_to_shared(&s_qw[buf][r * 3 + cc][lane]);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst),
                             "l"(qcol + (int64_t)(i + r) * p.pitch + cc * cs) : "memory");
            }
    };
#pragma unroll
    for (int d = 0; d < RDEPTH - 1; ++d) {
        if (r0 + 2 * d < r1) prefetch(r0 + 2 * d, d);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    const int j0 = __ldg(a.axis_i + coloff + j);
    double wy[2], uy[2];
    int ja[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        wy[e] = __ldg(a.axis_w + coloff + j + e);
        uy[e] = 1.0 - wy[e];
        ja[e] = a.axis_dry ? __ldg(a.axis_dry + coloff + j + e) : 0;
    }
    unsigned off[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) off[c] = (unsigned)(((int64_t)c * plane + j0) * 8);
    const int64_t rowbytes = nya * 8;

    auto corners = [&](double (&C)[3][4], int n, int64_t rowb) {
        const char* b0 = s_base[n] + rowb;
        const char* b1 = b0 + rowbytes;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double* q0 = reinterpret_cast<const double*>(b0 + off[c]);
            const double* q1 = reinterpret_cast<const double*>(b1 + off[c]);
            C[c][0] = __ldg(q0); C[c][1] = __ldg(q1); C[c][2] = __ldg(q0 + 1); C[c][3] = __ldg(q1 + 1);
        }
    };
    unsigned long long cnt = 0;
    int buf = 0;
    int i0n = __ldg(a.axis_i + rowoff + r0);
    double wxn[2] = {__ldg(a.axis_w + rowoff + r0), __ldg(a.axis_w + rowoff + r0 + 1)};
    for (unsigned i = r0; i < r1; i += 2, buf = buf + 1 == RDEPTH ? 0 : buf + 1) {
        if (i + 2 * (RDEPTH - 1) < r1) prefetch(i + 2 * (RDEPTH - 1), buf == 0 ? RDEPTH - 1 : buf - 1);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        const int64_t rowb = (int64_t)i0n * rowbytes;
        double wx[2] = {wxn[0], wxn[1]}, ux[2];
        ux[0] = 1.0 - wx[0]; ux[1] = 1.0 - wx[1];
        double C0[3][4], C1[3][4], C2[3][4];
        corners(C0, 0, rowb);
        if (K3_QUAD_DEPTH > 2 && nidx > 1) corners(C1, 1, rowb);
        if (i + 2 < r1) {   // the next row pair's stencil row and weights
            i0n = __ldg(a.axis_i + rowoff + i + 2);
            wxn[0] = __ldg(a.axis_w + rowoff + i + 2); wxn[1] = __ldg(a.axis_w + rowoff + i + 3);
        }
        double W[2][2][4];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                W[r][e][0] = ux[r] * uy[e]; W[r][e][1] = wx[r] * uy[e];
                W[r][e][2] = ux[r] * wy[e]; W[r][e][3] = wx[r] * wy[e];
            }
        asm volatile("cp.async.wait_group %0;\n" ::"n"(RDEPTH - 1) : "memory");
        __syncwarp();
        double q[2][2][3];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double2 v = s_qw[buf][r * 3 + c][lane];
                q[r][0][c] = v.x; q[r][1][c] = v.y;
            }
        __syncwarp();
        double best[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        auto accumulate = [&](const double (&C)[3][4]) {
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    double d = 0.0;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double qh = corner_interp<FASTW>(C[c][0], C[c][1], C[c][2], C[c][3], ux[r], uy[e],
                                                               wx[r], wy[e], W[r][e]);
                        d = c == 0 ? qh * q[r][e][c] : (FASTW ? fma(qh, q[r][e][c], d) : d + qh * q[r][e][c]);
                    }
                    best[r][e] = fmax(best[r][e], fabs(d));
                }
        };
        if (K3_QUAD_DEPTH > 2) {                 // snapshots n+1, n+2 in flight during n's arithmetic
            for (int n = 0; n < nidx; n += 3) {
                if (n + 2 < nidx) corners(C2, n + 2, rowb);
                accumulate(C0);
                if (n + 1 >= nidx) break;
                if (n + 3 < nidx) corners(C0, n + 3, rowb);
                accumulate(C1);
                if (n + 2 >= nidx) break;
                if (n + 4 < nidx) corners(C1, n + 4, rowb);
                accumulate(C2);
            }
        } else {
            for (int n = 0; n < nidx; n += 2) {      // snapshot n+1's corners load during n's arithmetic
                if (n + 1 < nidx) corners(C1, n + 1, rowb);
                accumulate(C0);
                if (n + 1 < nidx) {
                    if (n + 2 < nidx) corners(C0, n + 2, rowb);
                    accumulate(C1);
                }
            }
        }
        (void)C2;
        unsigned bits = 0;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (a.swe) {   // forward dry cells
                const double* cp = a.aux + a.aux_stride + p.offset + (int64_t)(i + r + g) * p.pitch + (j + g);
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (!(__ldg(cp + e) > 0.0)) best[r][e] = 0.0;
            }
            if (a.adj_wet != nullptr && a.axis_dry) {   // adjoint cell containing the centre is dry
                const int ia = __ldg(a.axis_dry + rowoff + i + r);
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (!a.adj_wet[(int64_t)ia * nya + ja[e]]) best[r][e] = 0.0;
            }
            const unsigned base = (i + r) * ny + seg * 64u;
            if (a.best != nullptr)
                *reinterpret_cast<double2*>(a.best + a.best_offset[pidx] + base + 2u * lane) =
                    make_double2(best[r][0], best[r][1]);
            bits |= (best[r][0] > a.tolerance ? 1u : 0u) << (2 * r) | (best[r][1] > a.tolerance ? 2u : 0u) << (2 * r);
        }
        // word (row r, half h), bit b = cell 32h + b of the row, held by lane 16h + b/2 as element b%2
        const unsigned t0 = __shfl_sync(0xffffffffu, bits, lane >> 1) >> (lane & 1);
        const unsigned t1 = __shfl_sync(0xffffffffu, bits, 16 + (lane >> 1)) >> (lane & 1);
        const unsigned w00 = __ballot_sync(0xffffffffu, t0 & 1u), w01 = __ballot_sync(0xffffffffu, t1 & 1u);
        const unsigned w10 = __ballot_sync(0xffffffffu, (t0 >> 2) & 1u), w11 = __ballot_sync(0xffffffffu, (t1 >> 2) & 1u);
        if (lane < 4) {
            const unsigned r = lane >> 1, h = lane & 1u;
            const unsigned wv = lane == 0 ? w00 : (lane == 1 ? w01 : (lane == 2 ? w10 : w11));
            a.flag_bits[p.flag_word + (((i + r) * ny + seg * 64u) >> 5) + h] = wv;
        }
        cnt += __popc(w00) + __popc(w01) + __popc(w10) + __popc(w11);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    if (lane == 0 && cnt) atomicAdd(&a.counts[pidx], cnt);
}

template <bool FASTW>
__global__ void __launch_bounds__(32 * K3_ROW_WARPS, FASTW ? K3_QUAD_MINB_FAST : K3_QUAD_MINB)
    k3_quad(AdjFlagArgs a, int run) {
    __shared__ const char* s_base[K3_MAXN];     // snapshot base addresses
    __shared__ double2 s_q[K3_ROW_WARPS][RDEPTH][6][32];
    {
        const int64_t snap_b = (int64_t)a.nxa * a.nya * 3 * 8;
        for (int n = threadIdx.x; n < a.nidx; n += blockDim.x)
            s_base[n] = reinterpret_cast<const char*>(a.ring) + (int64_t)a.snap_index[n] * snap_b;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned r0 = blockIdx.x * (unsigned)run;               // run is even
    quad_rows<FASTW>(a, s_base, s_q[warp], blockIdx.z, blockIdx.y * K3_ROW_WARPS + warp, r0, r0 + (unsigned)run,
                     lane);
}

// Bound pass of a pruned window: one warp per 64-column segment and a run of
// row pairs of the quad layout (the blocks k3_quad's warps own).  Per block the
// cells' bounds sum_c |q_c| E_c, E_c the maximum of the node envelope
// (AdjFlagArgs.envelope, k3_envelope) over the cell's bilinear stencil; a
// block none of whose cells can exceed the tolerance
// gets zero flag words, the others go to the work list for k3_quad_list.
// Loads of the next row pair are issued before this one's bound is formed.
__global__ void __launch_bounds__(256) k3_bound(AdjFlagArgs a, int run) {
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int pidx = blockIdx.z;
    const AdjPatch p = a.patches[pidx];
    const unsigned nseg = (unsigned)p.ny / 64u;
    const unsigned seg = (unsigned)warp % (nseg ? nseg : 1u), chunk = (unsigned)warp / (nseg ? nseg : 1u);
    const unsigned r0 = chunk * (unsigned)run;
    if (nseg == 0 || r0 >= (unsigned)p.nx) return;
    const unsigned r1 = min(r0 + (unsigned)run, (unsigned)p.nx);
    const unsigned ny = (unsigned)p.ny, j = seg * 64u + 2u * lane;
    const int64_t nya = a.nya, plane = (int64_t)a.nxa * nya, cs = a.comp_stride;
    const int64_t rowoff = a.axis_off[2 * pidx], coloff = a.axis_off[2 * pidx + 1];
    // node envelope; the stencil maximum over the 2 x 2 nodes is taken here (the clamped
    // stencil of interpolate_uniform never passes the last row / column)
    const double* env = a.envelope + __ldg(a.axis_i + coloff + j);
    const double* qc = a.q + p.offset + (int64_t)a.ghost * p.pitch + a.ghost + j;
    const double tol = a.tolerance;
    double2 Q[2][3];
    double E[3];
    auto load = [&](unsigned i) {
        const int64_t eo = (int64_t)__ldg(a.axis_i + rowoff + i) * nya;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double* e = env + c * plane + eo;
            E[c] = nanmax(nanmax(__ldg(e), __ldg(e + 1)), nanmax(__ldg(e + nya), __ldg(e + nya + 1)));
#pragma unroll
            for (int r = 0; r < 2; ++r)
                Q[r][c] = __ldcs(reinterpret_cast<const double2*>(qc + (int64_t)(i + r) * p.pitch + c * cs));
        }
    };
    load(r0);
    for (unsigned i = r0; i < r1; i += 2) {
        double2 q[2][3];
        double e[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) { e[c] = E[c]; q[0][c] = Q[0][c]; q[1][c] = Q[1][c]; }
        if (i + 2 < r1) load(i + 2);
        bool need = false;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            // |d| <= (1 + 12u) sum_c |q_c| E_c for every snapshot of the window (bilinear and
            // time-linear weights in [0, 1]); the 1e-12 margin covers that and this sum's rounding
            const double b0 = fma(fabs(q[r][2].x), e[2], fma(fabs(q[r][1].x), e[1], fabs(q[r][0].x) * e[0]));
            const double b1 = fma(fabs(q[r][2].y), e[2], fma(fabs(q[r][1].y), e[1], fabs(q[r][0].y) * e[0]));
            need |= !(b0 * (1.0 + 1e-12) <= tol) || !(b1 * (1.0 + 1e-12) <= tol);
        }
        if (__any_sync(0xffffffffu, need)) {
            if (lane == 0) {
                const int k = atomicAdd(a.work, 1);
                reinterpret_cast<int4*>(a.work)[1 + k] = make_int4(pidx, (int)seg, (int)i, 0);
            }
        } else if (lane < 4) {
            const unsigned r = lane >> 1, h = lane & 1u;
            a.flag_bits[p.flag_word + (((i + r) * ny + seg * 64u) >> 5) + h] = 0u;
        }
    }
}

// Pruned windows (AdjFlagArgs.envelope): k3_bound streamed every row pair of
// the quad layout once and wrote zero flag words where no cell of the warp's
// 2 x 64 block can reach the tolerance; the remaining blocks, listed in
// work[2 ..] as (patch, segment, row pair), are evaluated here by persistent
// warps pulling from the list (the unpruned blocks cluster where the wave and
// the adjoint overlap, so a static split would leave most warps idle).
template <bool FASTW>
__global__ void __launch_bounds__(32 * K3_ROW_WARPS, FASTW ? K3_QUAD_MINB_FAST : K3_QUAD_MINB)
    k3_quad_list(AdjFlagArgs a) {
    __shared__ const char* s_base[K3_MAXN];
    __shared__ double2 s_q[K3_ROW_WARPS][RDEPTH][6][32];
    __shared__ int s_item[K3_ROW_WARPS];
    {
        const int64_t snap_b = (int64_t)a.nxa * a.nya * 3 * 8;
        for (int n = threadIdx.x; n < a.nidx; n += blockDim.x)
            s_base[n] = reinterpret_cast<const char*>(a.ring) + (int64_t)a.snap_index[n] * snap_b;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int count = __ldcg(a.work);
    for (;;) {
        if (lane == 0) s_item[warp] = atomicAdd(a.work + 1, 1);
        __syncwarp();
        const int it = s_item[warp];
        __syncwarp();
        if (it >= count) break;
        const int4 w = __ldcg(reinterpret_cast<const int4*>(a.work) + 1 + it);
        quad_rows<FASTW>(a, s_base, s_q[warp], w.x, (unsigned)w.y, (unsigned)w.z, (unsigned)w.z + 2u, lane);
    }
}

// ---------------------------------------------------------------------------
// Mode-0 windows when every weight is exactly 0 or 1 (ADJ_FLAG_DIRECT, e.g.
// the C3 forward and adjoint grids coincide): the reference's bilinear
// expression C00 ux uy + C10 wx uy + C01 ux wy + C11 wx wy reduces to the one
// corner whose weights are 1 (the others contribute signed zeros), so each
// cell-snapshot is one adjoint value per component -- bitwise equal for
// finite adjoint fields.  Lane l owns columns j + 32kk (coalesced adjoint
// loads); the next snapshot's values load while this one's dot products run.
template <int NCD>
__global__ void __launch_bounds__(32 * K3_ROW_WARPS, 3) k3_direct(AdjFlagArgs a, int run) {
    __shared__ const char* s_base[K3_MAXN];
    const int nidx = a.nidx;
    {
        const int64_t snap_b = (int64_t)a.nxa * a.nya * 3 * 8;
        for (int n = threadIdx.x; n < nidx; n += blockDim.x)
            s_base[n] = reinterpret_cast<const char*>(a.ring) + (int64_t)a.snap_index[n] * snap_b;
    }
    __syncthreads();
    const int pidx = blockIdx.z;
    const AdjPatch p = a.patches[pidx];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned seg = blockIdx.y * K3_ROW_WARPS + warp;
    const unsigned nseg = (unsigned)p.ny / (32u * NCD);
    const unsigned r0 = blockIdx.x * (unsigned)run;
    if (seg >= nseg || r0 >= (unsigned)p.nx) return;               // warp-uniform; no barrier below
    const unsigned r1 = min(r0 + (unsigned)run, (unsigned)p.nx);
    const unsigned ny = (unsigned)p.ny, j = seg * (32u * NCD) + lane;
    const int g = a.ghost;
    const int64_t cs = a.comp_stride;
    const int64_t nya = a.nya;
    const int64_t plane_b = (int64_t)a.nxa * nya * 8;
    const int64_t rowoff = a.axis_off[2 * pidx], coloff = a.axis_off[2 * pidx + 1];
    unsigned coff[NCD];   // byte offset of this lane's adjoint column (j0 + the unit weight)
    int ja[NCD];
#pragma unroll
    for (int kk = 0; kk < NCD; ++kk) {
        const int jt = (int)(j + 32 * kk);
        coff[kk] = (unsigned)((__ldg(a.axis_i + coloff + jt) + (__ldg(a.axis_w + coloff + jt) > 0.5 ? 1 : 0)) * 8);
        ja[kk] = a.axis_dry ? __ldg(a.axis_dry + coloff + jt) : 0;
    }
    unsigned long long cnt = 0;
    for (unsigned i = r0; i < r1; ++i) {
        const int64_t rowb = (int64_t)(__ldg(a.axis_i + rowoff + i) + (__ldg(a.axis_w + rowoff + i) > 0.5 ? 1 : 0)) *
                             nya * 8;
        const double* qr = a.q + p.offset + (int64_t)(i + g) * p.pitch + g + j;
        double q[NCD][3];
#pragma unroll
        for (int kk = 0; kk < NCD; ++kk)
#pragma unroll
            for (int c = 0; c < 3; ++c) q[kk][c] = __ldcs(qr + c * cs + 32 * kk);   // streamed once
        double V0[NCD][3], V1[NCD][3];
        auto load = [&](double (&V)[NCD][3], int n) {
            const char* b = s_base[n] + rowb;
#pragma unroll
            for (int kk = 0; kk < NCD; ++kk)
#pragma unroll
                for (int c = 0; c < 3; ++c) V[kk][c] = __ldg(reinterpret_cast<const double*>(b + c * plane_b + coff[kk]));
        };
        double best[NCD];
#pragma unroll
        for (int kk = 0; kk < NCD; ++kk) best[kk] = 0.0;
        auto accumulate = [&](const double (&V)[NCD][3]) {
#pragma unroll
            for (int kk = 0; kk < NCD; ++kk) {
                double d = 0.0;
#pragma unroll
                for (int c = 0; c < 3; ++c) d = c == 0 ? V[kk][c] * q[kk][c] : d + V[kk][c] * q[kk][c];
                best[kk] = fmax(best[kk], fabs(d));
            }
        };
        if (nidx > 0) load(V0, 0);   // empty window (t past the last snapshot): best stays 0
        for (int n = 0; n < nidx; n += 2) {
            if (n + 1 < nidx) load(V1, n + 1);
            accumulate(V0);
            if (n + 1 < nidx) {
                if (n + 2 < nidx) load(V0, n + 2);
                accumulate(V1);
            }
        }
        if (a.swe) {   // forward dry cells
            const double* cp = a.aux + a.aux_stride + p.offset + (int64_t)(i + g) * p.pitch + (j + g);
#pragma unroll
            for (int kk = 0; kk < NCD; ++kk)
                if (!(__ldg(cp + 32 * kk) > 0.0)) best[kk] = 0.0;
        }
        if (a.adj_wet != nullptr && a.axis_dry) {
            const int ia = __ldg(a.axis_dry + rowoff + i);
#pragma unroll
            for (int kk = 0; kk < NCD; ++kk)
                if (!a.adj_wet[(int64_t)ia * nya + ja[kk]]) best[kk] = 0.0;
        }
        const unsigned base = i * ny + seg * (32u * NCD);
#pragma unroll
        for (int kk = 0; kk < NCD; ++kk) {
            if (a.best != nullptr) a.best[a.best_offset[pidx] + base + 32u * kk + lane] = best[kk];
            const unsigned word = __ballot_sync(0xffffffffu, best[kk] > a.tolerance);
            if (lane == 0) a.flag_bits[p.flag_word + ((base >> 5) + kk)] = word;
            cnt += __popc(word);
        }
    }
    if (lane == 0 && cnt) atomicAdd(&a.counts[pidx], cnt);
}

// ADJAMR_K3_PAIRS=0 selects the one-cell-per-lane table kernel (A/B measurements)
static bool k3_pairs() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("ADJAMR_K3_PAIRS");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// ADJAMR_K3_DIRECT=0 disables the direct (unit-weight) kernel (A/B measurements)
static bool k3_direct_on() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("ADJAMR_K3_DIRECT");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// rows per warp of k3_direct: the grid about one wave of resident CTAs
static int k3_direct_run(const AdjFlagArgs& a) {
    static int res = 0;
    if (res == 0) {
        int per_sm = 0, dev = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_direct<4>, 32 * K3_ROW_WARPS, 0);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        res = (per_sm < 1 ? 1 : per_sm) * sms;
    }
    const int64_t segs = ((int64_t)a.max_cols / 128 + K3_ROW_WARPS - 1) / K3_ROW_WARPS;
    int64_t runs = res / (segs * a.npatch > 0 ? segs * a.npatch : 1);
    if (runs < 1) runs = 1;
    const int64_t run = (a.max_rows + runs - 1) / runs;
    return (int)(run < 1 ? 1 : run);
}

// ADJAMR_K3_QUAD=0 disables the quad kernel for multi-snapshot windows (A/B measurements)
static bool k3_quad_on() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("ADJAMR_K3_QUAD");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// ADJAMR_K3_QUAD1=1 also routes single-snapshot windows to k3_quad (A/B measurements)
static bool k3_quad1() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("ADJAMR_K3_QUAD1");
        on = (e && e[0] == '1') ? 1 : 0;
    }
    return on == 1;
}

// rows per warp of k3_quad: even, and the grid about one wave of resident CTAs
static int k3_quad_run(const AdjFlagArgs& a) {
    static int resident[2] = {0, 0};
    const bool fw = a.variant == ADJ_VARIANT_FAST;
    int& res = resident[fw ? 1 : 0];
    if (res == 0) {
        int per_sm = 0, dev = 0, sms = 0;
        if (fw) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_quad<true>, 32 * K3_ROW_WARPS, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_quad<false>, 32 * K3_ROW_WARPS, 0);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        res = (per_sm < 1 ? 1 : per_sm) * sms;
    }
    const int64_t segs = ((int64_t)a.max_cols / 64 + K3_ROW_WARPS - 1) / K3_ROW_WARPS;
    int64_t runs = res / (segs * a.npatch > 0 ? segs * a.npatch : 1);
    if (runs < 1) runs = 1;
    int64_t run = (a.max_rows + runs - 1) / runs;
    run += run & 1;
    return (int)(run < 2 ? 2 : run);
}

// ADJAMR_K3_ROWP=0 disables the paired row kernel (A/B measurements)
static bool k3_rowp_on() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("ADJAMR_K3_ROWP");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// ADJAMR_K3_ROW=0 disables the row-layout kernel (A/B measurements)
static bool k3_row_on() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("ADJAMR_K3_ROW");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// Rows per warp of k3_row: K3_ROW_RUN, or (0) the run that makes the grid
// about one wave of resident CTAs, so each warp's column tables and pipeline
// fill amortise over as many rows as the device allows.
static int k3_row_run(const AdjFlagArgs& a, bool m1, bool pairs) {
    if (K3_ROW_RUN > 0) return K3_ROW_RUN;
    static int resident[3] = {0, 0, 0};
    int& res = resident[pairs ? 2 : (m1 ? 1 : 0)];
    if (res == 0) {
        int per_sm = 0, dev = 0, sms = 0;
        if (pairs) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_rowp, 32 * K3_ROW_WARPS, 0);
        else if (m1) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_row<true>, 32 * K3_ROW_WARPS, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_row<false>, 32 * K3_ROW_WARPS, 0);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        res = (per_sm < 1 ? 1 : per_sm) * sms;
    }
    const int64_t segs = ((int64_t)a.max_cols / (32 * RNC) + K3_ROW_WARPS - 1) / K3_ROW_WARPS;
    const int64_t ctas_per_run_row = segs * a.npatch;          // CTAs per row-run index
    int64_t runs = res / (ctas_per_run_row > 0 ? ctas_per_run_row : 1);
    if (runs < 1) runs = 1;
    int64_t run = (a.max_rows + runs - 1) / runs;
    if (run < 4) run = 4;
    return (int)run;
}

int flag_adjoint(const AdjFlagArgs& a) {
    if (a.npatch <= 0 || a.max_cells <= 0) return ADJ_OK;
    const int threads = 256;
    const int64_t bx = ((int64_t)a.max_cells + threads * NC - 1) / (threads * NC);
    dim3 grid((unsigned)bx, (unsigned)a.npatch);
    cudaStream_t st = (cudaStream_t)a.stream;
    const bool tab = a.axis_w && a.axis_i && a.axis_off;
    if (tab && a.nidx <= K3_MAXN && !(a.ndim == 2 && a.adj_wet && !a.axis_dry)) {
        const bool m1 = a.mode == 1;
        if (a.ndim == 1 && a.m == 2) {
            if (m1) k3_flag_t<2, false, true><<<grid, threads, 0, st>>>(a);
            else k3_flag_t<2, false, false><<<grid, threads, 0, st>>>(a);
        } else if (a.ndim == 2 && a.m == 3) {
            // pairs pay off once a window has several snapshots (measured: 1.37 vs 1.69 ms at
            // 21 snapshots on C4; 0.23 vs 0.22 ms at one)
            if (!m1 && a.nidx >= 1 && (a.layout & ADJ_FLAG_ROWS) && (a.layout & ADJ_FLAG_DIRECT) && k3_direct_on() &&
                (int64_t)a.nxa * a.nya * 3 * 8 < (int64_t(1) << 32)) {
                const int run = k3_direct_run(a);
                const dim3 gr((unsigned)((a.max_rows + run - 1) / run),
                              (unsigned)((a.max_cols / 128 + K3_ROW_WARPS - 1) / K3_ROW_WARPS), (unsigned)a.npatch);
                k3_direct<4><<<gr, 32 * K3_ROW_WARPS, 0, st>>>(a, run);
            } else if (!m1 && a.nidx >= (k3_quad1() ? 1 : 2) && (a.layout & ADJ_FLAG_ROWS) && (a.layout & ADJ_FLAG_QUADS) &&
                k3_quad_on() &&
                (int64_t)a.nxa * a.nya * 3 * 8 < (int64_t(1) << 32)) {
                const int run = k3_quad_run(a);
                const dim3 gr((unsigned)((a.max_rows + run - 1) / run),
                              (unsigned)((a.max_cols / 64 + K3_ROW_WARPS - 1) / K3_ROW_WARPS), (unsigned)a.npatch);
                if (a.envelope && a.work && !a.best && a.tolerance > 1e-280) {
                    // pruned window: envelope, bound pass + work list, listed blocks only
                    const int64_t nodes = (int64_t)a.nxa * a.nya;
                    const int eb = (int)((nodes + 255) / 256 < 148 * 16 ? (nodes + 255) / 256 : 148 * 16);
                    int rc = record_cuda(cudaMemsetAsync(a.work, 0, 2 * sizeof(int32_t), st), "memset work");
                    if (rc) return rc;
                    k3_envelope<<<eb, 256, 0, st>>>(a);
                    constexpr int BRUN = 16;   // rows per bound warp (8 row pairs)
                    const int64_t warps = (int64_t)(a.max_cols / 64) * ((a.max_rows + BRUN - 1) / BRUN);
                    k3_bound<<<dim3((unsigned)((warps + 7) / 8), 1, (unsigned)a.npatch), 256, 0, st>>>(a, BRUN);
                    static int list_ctas[2] = {0, 0};
                    const bool fw = a.variant == ADJ_VARIANT_FAST;
                    if (!list_ctas[fw]) {
                        int per_sm = 0, dev = 0, sms = 0;
                        if (fw) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_quad_list<true>, 32 * K3_ROW_WARPS, 0);
                        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_quad_list<false>, 32 * K3_ROW_WARPS, 0);
                        cudaGetDevice(&dev);
                        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                        list_ctas[fw] = (per_sm < 1 ? 1 : per_sm) * sms;
                    }
                    if (fw) k3_quad_list<true><<<list_ctas[1], 32 * K3_ROW_WARPS, 0, st>>>(a);
                    else k3_quad_list<false><<<list_ctas[0], 32 * K3_ROW_WARPS, 0, st>>>(a);
                } else if (a.variant == ADJ_VARIANT_FAST) {
                    k3_quad<true><<<gr, 32 * K3_ROW_WARPS, 0, st>>>(a, run);
                } else {
                    k3_quad<false><<<gr, 32 * K3_ROW_WARPS, 0, st>>>(a, run);
                }
            } else if (k3_pairs() && a.nidx >= 2) {
                const bool fw = a.variant == ADJ_VARIANT_FAST;
                if (m1 && fw) k3_pair<true, true><<<grid, threads, 0, st>>>(a);
                else if (m1) k3_pair<true, false><<<grid, threads, 0, st>>>(a);
                else if (fw) k3_pair<false, true><<<grid, threads, 0, st>>>(a);
                else k3_pair<false, false><<<grid, threads, 0, st>>>(a);
            } else if (a.nidx == 1 && (a.layout & ADJ_FLAG_ROWS) && k3_row_on()) {
                // (row runs, column segments / warps per CTA, patches); max_rows = the tallest patch
                const bool pairs = !m1 && (a.layout & ADJ_FLAG_PAIRS) && k3_rowp_on() &&
                                   (int64_t)a.nxa * a.nya * 3 * 8 < (int64_t(1) << 32);   // 32-bit corner offsets
                const int run = k3_row_run(a, m1, pairs);
                const dim3 gr((unsigned)((a.max_rows + run - 1) / run),
                              (unsigned)((a.max_cols / (32 * RNC) + K3_ROW_WARPS - 1) / K3_ROW_WARPS),
                              (unsigned)a.npatch);
                if (pairs) k3_rowp<<<gr, 32 * K3_ROW_WARPS, 0, st>>>(a, run);
                else if (m1) k3_row<true><<<gr, 32 * K3_ROW_WARPS, 0, st>>>(a, run);
                else k3_row<false><<<gr, 32 * K3_ROW_WARPS, 0, st>>>(a, run);
            } else {
                if (m1) k3_flag_t<3, true, true><<<grid, threads, 0, st>>>(a);
                else k3_flag_t<3, true, false><<<grid, threads, 0, st>>>(a);
            }
        } else {
            return ADJ_ERR_BAD_ARG;
        }
        return check_launch("k3_flag_t");
    }
    if (a.ndim == 1) {
        if (a.m != 2) return ADJ_ERR_BAD_ARG;
        if (tab) k3_flag<2, false, true><<<grid, threads, 0, st>>>(a);
        else k3_flag<2, false, false><<<grid, threads, 0, st>>>(a);
    } else {
        if (a.m != 3) return ADJ_ERR_BAD_ARG;
        if (tab) k3_flag<3, true, true><<<grid, threads, 0, st>>>(a);
        else k3_flag<3, true, false><<<grid, threads, 0, st>>>(a);
    }
    return check_launch("k3_flag");
}

// ---------------------------------------------------------------------------
// evaluate_J: signed inner products over uncovered cells, per-block sums.

__global__ void k3_cover(AdjFunctionalArgs a) {
    const AdjPatch f = a.finer[blockIdx.y];
    const int r = a.ratio;
    const int ci0 = f.lo_x / r, ci1 = (f.lo_x + f.nx - 1) / r;
    const int cj0 = a.ndim == 2 ? f.lo_y / r : 0, cj1 = a.ndim == 2 ? (f.lo_y + f.ny - 1) / r : 0;
    const int nj = cj1 - cj0 + 1;
    const int n = (ci1 - ci0 + 1) * nj;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int i = ci0 + t / nj, j = cj0 + t % nj;
        if (i < a.level_nx && j < a.level_ny) a.covered[(int64_t)i * a.level_ny + j] = 1;
    }
}

template <int M, bool TWO_D>
__global__ void __launch_bounds__(256) k3_functional(AdjFunctionalArgs a) {
    __shared__ double s_part[8];
    const int pidx = blockIdx.y;
    const AdjPatch p = a.patches[pidx];
    const int ny = TWO_D ? p.ny : 1;
    const int ncell = p.nx * ny;
    const int g = a.ghost, gy = TWO_D ? g : 0;
    const unsigned plane = (unsigned)a.nxa * (unsigned)a.nya;
    double acc = 0.0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ncell; t += a.blocks_x * blockDim.x) {
        const int i = t / ny, j = t - (t / ny) * ny;
        if (a.covered && a.covered[(int64_t)(p.lo_x + i) * a.level_ny + (TWO_D ? p.lo_y + j : 0)]) continue;
        const int64_t o = p.offset + (int64_t)(i + g) * p.pitch + (j + gy);
        // cell centre (PatchSpec.cell_centers) and interpolate_uniform's bounds check
        const double x = a.origin_x + ((p.lo_x + i) + 0.5) * a.dx;
        const double y = TWO_D ? a.origin_y + ((p.lo_y + j) + 0.5) * a.dy : 0.0;
        const double hx = a.a_origin_x + a.nxa * a.a_dx;
        const double eps = 1e-12 * fmax(fabs(hx - a.a_origin_x), 1.0);
        bool oob = (x < a.a_origin_x - eps) || (x > hx + eps);
        if (TWO_D) {
            const double hy = a.a_origin_y + a.nya * a.a_dy;
            oob |= (y < a.a_origin_y - eps) || (y > hy + eps);
        }
        if (oob) atomicOr(a.status, 1);
        int i0, j0 = 0;
        double wx, wy = 0.0;
        uweights(x, a.a_origin_x, a.a_dx, a.nxa, &i0, &wx);
        if (TWO_D) uweights(y, a.a_origin_y, a.a_dy, a.nya, &j0, &wy);
        const int i1 = min(i0 + 1, a.nxa - 1);
        const int j1 = TWO_D ? min(j0 + 1, a.nya - 1) : 0;
        const unsigned o00 = (unsigned)i0 * a.nya + j0, o10 = (unsigned)i1 * a.nya + j0;
        const unsigned o01 = (unsigned)i0 * a.nya + j1, o11 = (unsigned)i1 * a.nya + j1;
        const double ux = 1.0 - wx, uy = 1.0 - wy;
        double dot = 0.0;
        const int k = a.snap;
#pragma unroll
        for (int c = 0; c < M; ++c) {
            double qh;
            if (k < 0) {
                const double* fc = a.ring + ((int64_t)(-k - 1) * M + c) * plane;
                qh = TWO_D ? fc[o00] * ux * uy + fc[o10] * wx * uy + fc[o01] * ux * wy + fc[o11] * wx * wy
                           : fc[o00] * ux + fc[o10] * wx;
            } else {   // interpolate_time, then the spatial stencil
                const double* ac = a.ring + ((int64_t)k * M + c) * plane;
                const double* bc = ac + (int64_t)plane * M;
                const double v00 = (1.0 - a.w) * ac[o00] + a.w * bc[o00];
                const double v10 = (1.0 - a.w) * ac[o10] + a.w * bc[o10];
                if (TWO_D) {
                    const double v01 = (1.0 - a.w) * ac[o01] + a.w * bc[o01];
                    const double v11 = (1.0 - a.w) * ac[o11] + a.w * bc[o11];
                    qh = v00 * ux * uy + v10 * wx * uy + v01 * ux * wy + v11 * wx * wy;
                } else {
                    qh = v00 * ux + v10 * wx;
                }
            }
            const double qc = a.q[c * a.comp_stride + o];
            dot = c == 0 ? qh * qc : dot + qh * qc;   // np.sum(qhat * q, axis=0)
        }
        acc = acc + dot;
    }
    // fixed-order block reduction
    for (int off = 16; off > 0; off >>= 1) acc = acc + __shfl_down_sync(0xffffffffu, acc, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_part[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = s_part[0];
        for (int wi = 1; wi < (int)(blockDim.x >> 5); ++wi) s = s + s_part[wi];
        a.partial[(int64_t)pidx * a.blocks_x + blockIdx.x] = s;
    }
}

int functional(const AdjFunctionalArgs& a) {
    cudaStream_t st = (cudaStream_t)a.stream;
    int rc = record_cuda(cudaMemsetAsync(a.status, 0, sizeof(int32_t), st), "memset status");
    if (rc) return rc;
    if (a.finer && a.nfiner > 0) {
        rc = record_cuda(cudaMemsetAsync(a.covered, 0, (size_t)a.level_nx * a.level_ny, st), "memset covered");
        if (rc) return rc;
        k3_cover<<<dim3(16, a.nfiner), 256, 0, st>>>(a);
        rc = check_launch("k3_cover");
        if (rc) return rc;
    }
    AdjFunctionalArgs b = a;
    if (!(a.finer && a.nfiner > 0)) b.covered = nullptr;
    const dim3 grid(a.blocks_x, a.npatch);
    if (a.ndim == 2 && a.m == 3) k3_functional<3, true><<<grid, 256, 0, st>>>(b);
    else if (a.ndim == 1 && a.m == 2) k3_functional<2, false><<<grid, 256, 0, st>>>(b);
    else return ADJ_ERR_BAD_ARG;
    return check_launch("k3_functional");
}

// gauges: interpolate_patch(interior_only=True), reference expression order
__global__ void k3_gauges(AdjGaugeArgs a) {
    const int gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= a.ngauge) return;
    const AdjGauge G = a.gauges[gi];
    for (int c = 0; c < a.m; ++c) {
        const double* d = a.q + c * a.comp_stride + G.base;
        double v;
        if (a.ndim == 1) {
            v = d[G.i0] * (1.0 - G.wx) + d[G.i1] * G.wx;
        } else {
            v = d[(int64_t)G.i0 * G.pitch + G.j0] * (1.0 - G.wx) * (1.0 - G.wy) +
                d[(int64_t)G.i1 * G.pitch + G.j0] * G.wx * (1.0 - G.wy) +
                d[(int64_t)G.i0 * G.pitch + G.j1] * (1.0 - G.wx) * G.wy +
                d[(int64_t)G.i1 * G.pitch + G.j1] * G.wx * G.wy;
        }
        a.out[gi * a.m + c] = v;
    }
}

int gauges(const AdjGaugeArgs& a) {
    if (a.ngauge <= 0) return ADJ_OK;
    k3_gauges<<<(a.ngauge + 127) / 128, 128, 0, (cudaStream_t)a.stream>>>(a);
    return check_launch("k3_gauges");
}

}  // namespace adj
