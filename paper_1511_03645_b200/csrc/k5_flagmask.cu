// K5: regrid flag post-processing on the device.
//
//   flag_cells region overrides      amr.py:137-154
//   buffer_flags (box dilation)      amr.py:157-179
//   level mask OR + nesting clip     amr.py:570-581, allowed_region_mask /
//                                    _erode geometry.py:341-368
//
// All boolean work: the result is exactly the reference's clipped mask.
#include "adj_common.cuh"

namespace adj {

// level occupancy: every parent patch marks its box
__global__ void k5_occupancy(AdjFlagMaskArgs a) {
    const AdjPatch p = a.patches[blockIdx.y];
    const int ny = a.ndim == 2 ? p.ny : 1;
    const int n = p.nx * ny;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int i = t / ny, j = t - (t / ny) * ny;
        a.occupancy[(int64_t)(p.lo_x + i) * a.level_ny + (p.lo_y + j)] = 1;
    }
}

// allowed = occupancy eroded by one cell, domain edges padded (np.pad 'edge')
__global__ void k5_allowed(AdjFlagMaskArgs a) {
    const int64_t total = (int64_t)a.level_nx * a.level_ny;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < total;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(c / a.level_ny), j = (int)(c - (c / a.level_ny) * a.level_ny);
        bool ok = true;
        for (int di = -1; di <= 1 && ok; ++di) {
            const int ii = min(max(i + di, 0), a.level_nx - 1);
            if (a.ndim == 2) {
                for (int dj = -1; dj <= 1; ++dj) {
                    const int jj = min(max(j + dj, 0), a.level_ny - 1);
                    ok = ok && a.occupancy[(int64_t)ii * a.level_ny + jj];
                }
            } else {
                ok = ok && a.occupancy[ii];
            }
        }
        a.mask[c] = ok ? 2 : 0;
    }
}

ADJ_D bool raw_flag(const AdjFlagMaskArgs& a, const AdjPatch& p, int ny, int rowoff, int coloff, int i, int j) {
    const int idx = i * ny + j;
    bool f = (a.flag_bits[p.flag_word + (idx >> 5)] >> (idx & 31)) & 1u;
    if (a.region_rows) {
        const unsigned in = (unsigned)a.region_rows[rowoff + i] & (a.ndim == 2 ? (unsigned)a.region_cols[coloff + j] : 0xffu);
        if (in & a.force_regions) f = true;
        if (in & a.clear_regions) f = false;
    }
    return f;
}

// buffered flags of every parent cell, clipped by the nesting mask
__global__ void k5_flags(AdjFlagMaskArgs a) {
    const AdjPatch p = a.patches[blockIdx.y];
    const int ny = a.ndim == 2 ? p.ny : 1;
    const int n = p.nx * ny;
    const int rowoff = a.region_rows ? a.region_row_off[blockIdx.y] : 0;
    const int coloff = a.region_cols ? a.region_col_off[blockIdx.y] : 0;
    const int b = a.buffer;
    unsigned long long cnt = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int i = t / ny, j = t - (t / ny) * ny;
        cnt += raw_flag(a, p, ny, rowoff, coloff, i, j) ? 1 : 0;
        bool any = false;
        const int i0 = max(i - b, 0), i1 = min(i + b, p.nx - 1);
        const int j0 = a.ndim == 2 ? max(j - b, 0) : 0, j1 = a.ndim == 2 ? min(j + b, ny - 1) : 0;
        for (int ii = i0; ii <= i1 && !any; ++ii)
            for (int jj = j0; jj <= j1 && !any; ++jj) any = raw_flag(a, p, ny, rowoff, coloff, ii, jj);
        if (any) {
            uint8_t* m = a.mask + (int64_t)(p.lo_x + i) * a.level_ny + (p.lo_y + j);
            if (*m & 2) *m = 3;
        }
    }
    // raw flag count (after region overrides)
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(a.raw_count, cnt);
}

int flag_level_mask(const AdjFlagMaskArgs& a) {
    cudaStream_t st = (cudaStream_t)a.stream;
    const int64_t total = (int64_t)a.level_nx * a.level_ny;
    int rc = record_cuda(cudaMemsetAsync(a.occupancy, 0, total, st), "memset occupancy");
    if (rc) return rc;
    rc = record_cuda(cudaMemsetAsync(a.raw_count, 0, sizeof(unsigned long long), st), "memset raw_count");
    if (rc) return rc;
    if (a.npatch <= 0) return record_cuda(cudaMemsetAsync(a.mask, 0, total, st), "memset mask");
    int bx = (a.max_cells + 255) / 256;
    if (bx > 1024) bx = 1024;
    k5_occupancy<<<dim3(bx, a.npatch), 256, 0, st>>>(a);
    rc = check_launch("k5_occupancy");
    if (rc) return rc;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k5_allowed<<<(int)blocks, 256, 0, st>>>(a);
    rc = check_launch("k5_allowed");
    if (rc) return rc;
    k5_flags<<<dim3(bx, a.npatch), 256, 0, st>>>(a);
    return check_launch("k5_flags");
}

}  // namespace adj
