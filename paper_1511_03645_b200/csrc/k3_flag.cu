// K3: adjoint inner-product flagging with bit-packed output.  Compiled with
// -fmad=false so the inner products are bitwise identical to the reference:
//   inner_product_field / inner_product_flags   adjoint.py:227-257
//   interpolate_uniform / _axis_weights         geometry.py:248-290
//   _adjoint_dry_at                             adjoint.py:217-224
//   AdjointSnapshotStore.interpolate_time       adjoint.py:98-110  (mode 1)
//
// One thread per forward interior cell; a warp covers 32 consecutive cells of
// one patch (row-major over the interior), so the warp's ballot is exactly
// one 32-bit flag word and its popcount the raw flagged count.
#include "adj_common.cuh"

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

template <int M, bool TWO_D>
__global__ void __launch_bounds__(256) k3_flag(AdjFlagArgs a) {
    const int pidx = blockIdx.y;
    const AdjPatch p = a.patches[pidx];
    const int64_t ncell = (int64_t)p.nx * p.ny;
    const int64_t cidx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t wbase = cidx & ~(int64_t)31;
    if (wbase >= ncell) return;  // whole warp beyond this patch
    const bool active = cidx < ncell;
    bool flag = false;
    if (active) {
        const int i = (int)(cidx / p.ny), j = (int)(cidx % p.ny);
        const int g = a.ghost;
        const int gy = TWO_D ? g : 0;
        const int64_t o = p.offset + (int64_t)(i + g) * p.pitch + (j + gy);
        double q[M];
#pragma unroll
        for (int c = 0; c < M; ++c) q[c] = a.q[c * a.comp_stride + o];
        // cell centre (PatchSpec.cell_centers, geometry.py:67-74)
        const double x = a.origin_x + ((p.lo_x + i) + 0.5) * a.dx;
        const double y = TWO_D ? a.origin_y + ((p.lo_y + j) + 0.5) * a.dy : 0.0;
        // bounds check of interpolate_uniform (geometry.py:271-283); the
        // reference derives eps from the x extent and applies it to both axes
        {
            const double hx = a.a_origin_x + a.nxa * a.a_dx;
            const double eps = 1e-12 * fmax(fabs(hx - a.a_origin_x), 1.0);
            bool oob = (x < a.a_origin_x - eps) || (x > hx + eps);
            if (TWO_D) {
                const double hy = a.a_origin_y + a.nya * a.a_dy;
                oob |= (y < a.a_origin_y - eps) || (y > hy + eps);
            }
            if (oob) atomicOr(a.status, 1);
        }
        int i0, j0 = 0; double wx, wy = 0.0;
        uweights(x, a.a_origin_x, a.a_dx, a.nxa, &i0, &wx);
        const int i1 = min(i0 + 1, a.nxa - 1);
        int j1 = 0;
        if (TWO_D) {
            uweights(y, a.a_origin_y, a.a_dy, a.nya, &j0, &wy);
            j1 = min(j0 + 1, a.nya - 1);
        }
        const int64_t plane = (int64_t)a.nxa * a.nya;
        const int64_t snap = plane * M;
        const int64_t o00 = (int64_t)i0 * a.nya + j0, o10 = (int64_t)i1 * a.nya + j0;
        const int64_t o01 = (int64_t)i0 * a.nya + j1, o11 = (int64_t)i1 * a.nya + j1;
        double best = 0.0;
        for (int n = 0; n < a.nidx; ++n) {
            const int k = a.snap_index[n];
            double dot = 0.0;
            if (a.mode == 0 || k < 0) {
                const int kk = k < 0 ? -k - 1 : k;
                const double* f = a.ring + kk * snap;
#pragma unroll
                for (int c = 0; c < M; ++c) {
                    const double* fc = f + c * plane;
                    double qh;
                    if (TWO_D)
                        qh = fc[o00] * (1.0 - wx) * (1.0 - wy) + fc[o10] * wx * (1.0 - wy) +
                             fc[o01] * (1.0 - wx) * wy + fc[o11] * wx * wy;
                    else
                        qh = fc[o00] * (1.0 - wx) + fc[o10] * wx;
                    dot = c == 0 ? qh * q[c] : dot + qh * q[c];
                }
            } else {
                // interpolate_time: vals = (1-w)*f[k] + w*f[k+1], then spatial interpolation
                const double w = a.interp_w[n];
                const double* fa = a.ring + k * snap;
                const double* fb = fa + snap;
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
                        qh = v00 * (1.0 - wx) * (1.0 - wy) + v10 * wx * (1.0 - wy) +
                             v01 * (1.0 - wx) * wy + v11 * wx * wy;
                    } else {
                        qh = v00 * (1.0 - wx) + v10 * wx;
                    }
                    dot = c == 0 ? qh * q[c] : dot + qh * q[c];
                }
            }
            best = fmax(best, fabs(dot));
        }
        if (a.swe && !(a.aux[a.aux_stride + o] > 0.0)) best = 0.0;   // forward dry cell
        if (TWO_D && a.adj_wet != nullptr) {
            // _adjoint_dry_at: astype(int) truncates toward zero, then clip
            int ia = (int)((x - a.a_origin_x) / a.a_dx);
            int ja = (int)((y - a.a_origin_y) / a.a_dy);
            ia = ia < 0 ? 0 : (ia > a.nxa - 1 ? a.nxa - 1 : ia);
            ja = ja < 0 ? 0 : (ja > a.nya - 1 ? a.nya - 1 : ja);
            if (!a.adj_wet[(int64_t)ia * a.nya + ja]) best = 0.0;
        }
        flag = best > a.tolerance;
        if (a.best != nullptr) a.best[a.best_offset[pidx] + cidx] = best;
    }
    const unsigned word = __ballot_sync(0xffffffffu, flag);
    if ((threadIdx.x & 31) == 0) {
        a.flag_bits[p.flag_word + (wbase >> 5)] = word;
        const int cnt = __popc(word);
        if (cnt) atomicAdd(&a.counts[pidx], (unsigned long long)cnt);
    }
}

int flag_adjoint(const AdjFlagArgs& a) {
    if (a.npatch <= 0 || a.max_cells <= 0) return ADJ_OK;
    const int threads = 256;
    const int64_t bx = ((int64_t)a.max_cells + threads - 1) / threads;
    dim3 grid((unsigned)bx, (unsigned)a.npatch);
    cudaStream_t st = (cudaStream_t)a.stream;
    if (a.ndim == 1) {
        if (a.m != 2) return ADJ_ERR_BAD_ARG;
        k3_flag<2, false><<<grid, threads, 0, st>>>(a);
    } else {
        if (a.m != 3) return ADJ_ERR_BAD_ARG;
        k3_flag<3, true><<<grid, threads, 0, st>>>(a);
    }
    return check_launch("k3_flag");
}

}  // namespace adj
