// Host-native signature-bisection clustering (the reference's cluster(),
// amr.py:186-337), identical boxes, for large level masks.
//
// Counts over any sub-box come from two prefix-sum tables (row-wise along y
// and column-wise along x), so bounding boxes, signatures and efficiencies
// cost O(perimeter) instead of O(area) per candidate box.  Tie-breaking,
// floating-point comparisons and the LIFO work order follow the reference.
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include <vector>
#include <algorithm>

#include "../../include/adjamr_b200.h"

namespace {

struct Mask {
    int nx, ny;                       // 1D: ny == 1
    std::vector<int32_t> rowp;        // rowp[i*(ny+1)+j] = sum_{j'<j} m[i][j']
    std::vector<int32_t> colp;        // colp[j*(nx+1)+i] = sum_{i'<i} m[i'][j]
    Mask(const uint8_t* m, int nx_, int ny_) : nx(nx_), ny(ny_), rowp((size_t)nx_ * (ny_ + 1)), colp((size_t)ny_ * (nx_ + 1)) {
        for (int i = 0; i < nx; ++i) {
            int32_t s = 0;
            rowp[(size_t)i * (ny + 1)] = 0;
            for (int j = 0; j < ny; ++j) { s += m[(size_t)i * ny + j] ? 1 : 0; rowp[(size_t)i * (ny + 1) + j + 1] = s; }
        }
        for (int j = 0; j < ny; ++j) {
            int32_t s = 0;
            colp[(size_t)j * (nx + 1)] = 0;
            for (int i = 0; i < nx; ++i) { s += m[(size_t)i * ny + j] ? 1 : 0; colp[(size_t)j * (nx + 1) + i + 1] = s; }
        }
    }
    // flagged cells of row i within columns [j0, j1]
    int32_t row(int i, int j0, int j1) const { return rowp[(size_t)i * (ny + 1) + j1 + 1] - rowp[(size_t)i * (ny + 1) + j0]; }
    // flagged cells of column j within rows [i0, i1]
    int32_t col(int j, int i0, int i1) const { return colp[(size_t)j * (nx + 1) + i1 + 1] - colp[(size_t)j * (nx + 1) + i0]; }
};

struct Box { int lo[2], hi[2]; };

// bounding box of the flags inside b; false when empty
bool bbox(const Mask& M, const Box& b, Box& out) {
    int i0 = -1, i1 = -1;
    for (int i = b.lo[0]; i <= b.hi[0]; ++i) if (M.row(i, b.lo[1], b.hi[1])) { i0 = i; break; }
    if (i0 < 0) return false;
    for (int i = b.hi[0]; i >= i0; --i) if (M.row(i, b.lo[1], b.hi[1])) { i1 = i; break; }
    int j0 = -1, j1 = -1;
    for (int j = b.lo[1]; j <= b.hi[1]; ++j) if (M.col(j, i0, i1)) { j0 = j; break; }
    for (int j = b.hi[1]; j >= j0; --j) if (M.col(j, i0, i1)) { j1 = j; break; }
    out.lo[0] = i0; out.hi[0] = i1; out.lo[1] = j0; out.hi[1] = j1;
    return true;
}

int64_t count(const Mask& M, const Box& b) {
    int64_t s = 0;
    for (int i = b.lo[0]; i <= b.hi[0]; ++i) s += M.row(i, b.lo[1], b.hi[1]);
    return s;
}

int64_t area(const Box& b) { return (int64_t)(b.hi[0] - b.lo[0] + 1) * (b.hi[1] - b.lo[1] + 1); }

void signature(const Mask& M, const Box& b, int axis, std::vector<int64_t>& sig) {
    sig.clear();
    if (axis == 0) for (int i = b.lo[0]; i <= b.hi[0]; ++i) sig.push_back(M.row(i, b.lo[1], b.hi[1]));
    else for (int j = b.lo[1]; j <= b.hi[1]; ++j) sig.push_back(M.col(j, b.lo[0], b.hi[0]));
}

struct Cut { int kind; int axis; int k; };   // kind 0 none, 1 hole, 2 edge

int argmax_shape(const Box& b, int nd) {
    int best = 0, n0 = b.hi[0] - b.lo[0] + 1;
    for (int a = 1; a < nd; ++a) if (b.hi[a] - b.lo[a] + 1 > n0) { best = a; n0 = b.hi[a] - b.lo[a] + 1; }
    return best;
}

Cut choose_cut(const Mask& M, const Box& b, int nd) {
    std::vector<int64_t> sig;
    bool have = false;
    double best_score = 0.0;
    int best_axis = 0, best_k = 0;
    for (int axis = 0; axis < nd; ++axis) {
        signature(M, b, axis, sig);
        const int n = (int)sig.size();
        const double mid = (n - 1) / 2.0;
        int k = -1;
        double dk = 0.0;
        for (int t = 0; t < n; ++t) {
            if (sig[t] != 0) continue;
            const double d = fabs(t - mid);
            if (k < 0 || d < dk) { k = t; dk = d; }
        }
        if (k >= 0) {
            const double score = fabs(k - mid) / (double)std::max(n, 1);
            if (!have || score < best_score) { have = true; best_score = score; best_axis = axis; best_k = k; }
        }
    }
    if (have) return Cut{1, best_axis, best_k};
    bool have_e = false;
    int64_t best_strength = 0;
    double best_negdist = 0.0;
    for (int axis = 0; axis < nd; ++axis) {
        signature(M, b, axis, sig);
        const int n = (int)sig.size();
        if (n < 4) continue;
        const double mid = (n - 1) / 2.0;
        for (int k = 0; k + 1 < n - 2; ++k) {
            const int64_t l0 = sig[k + 2] - 2 * sig[k + 1] + sig[k];
            const int64_t l1 = sig[k + 3] - 2 * sig[k + 2] + sig[k + 1];
            if ((l0 < 0 && l1 > 0) || (l0 > 0 && l1 < 0)) {
                const int64_t strength = l1 > l0 ? l1 - l0 : l0 - l1;
                const double negdist = -fabs((k + 1.5) - mid);
                if (!have_e || strength > best_strength || (strength == best_strength && negdist > best_negdist)) {
                    have_e = true; best_strength = strength; best_negdist = negdist; best_axis = axis; best_k = k + 1;
                }
            }
        }
    }
    if (have_e) return Cut{2, best_axis, best_k};
    const int axis = argmax_shape(b, nd);
    const int n = b.hi[axis] - b.lo[axis] + 1;
    if (n < 2) return Cut{0, 0, 0};
    return Cut{2, axis, n / 2 - 1};
}

int children(const Box& b, const Cut& c, Box* kids) {
    Box a = b, d = b;
    const int ax = c.axis;
    if (c.kind == 1) { a.hi[ax] = b.lo[ax] + c.k - 1; d.lo[ax] = b.lo[ax] + c.k + 1; }
    else { a.hi[ax] = b.lo[ax] + c.k; d.lo[ax] = b.lo[ax] + c.k + 1; }
    int n = 0;
    if (a.hi[ax] >= a.lo[ax]) kids[n++] = a;
    if (d.hi[ax] >= d.lo[ax]) kids[n++] = d;
    return n;
}

double tight_eff(const Mask& M, const Box& b) {
    Box bb;
    if (!bbox(M, b, bb)) return 1.0;
    return (double)count(M, bb) / (double)area(bb);
}

}  // namespace

extern "C" int adj_cluster(const uint8_t* mask, int ndim, int nx, int ny, double efficiency, int max_edge,
                           int32_t* boxes, double* effs, int max_boxes, int32_t* nboxes) {
    if (!mask || !boxes || !effs || !nboxes || nx < 1 || ny < 1 || (ndim != 1 && ndim != 2)) return ADJ_ERR_BAD_ARG;
    if (!(efficiency > 0.0 && efficiency <= 1.0)) return ADJ_ERR_BAD_ARG;
    const int nd = ndim;
    Mask M(mask, nx, ndim == 2 ? ny : 1);
    int n_out = 0;
    Box all{{0, 0}, {nx - 1, (ndim == 2 ? ny : 1) - 1}};
    Box top;
    *nboxes = 0;
    if (!bbox(M, all, top)) return ADJ_OK;
    std::vector<Box> stack{top};
    auto emit = [&](const Box& b, double eff) -> bool {
        if (n_out >= max_boxes) return false;
        boxes[4 * n_out + 0] = b.lo[0]; boxes[4 * n_out + 1] = b.lo[1];
        boxes[4 * n_out + 2] = b.hi[0]; boxes[4 * n_out + 3] = b.hi[1];
        effs[n_out] = eff;
        ++n_out;
        return true;
    };
    while (!stack.empty()) {
        Box b = stack.back();
        stack.pop_back();
        Box bb;
        if (!bbox(M, b, bb)) continue;
        const double eff = (double)count(M, bb) / (double)area(bb);
        int maxdim = 0;
        for (int a = 0; a < nd; ++a) maxdim = std::max(maxdim, bb.hi[a] - bb.lo[a] + 1);
        const bool oversize = max_edge > 0 && maxdim > max_edge;
        if (eff >= efficiency && !oversize) {
            if (eff < 1.0) {
                const Cut c = choose_cut(M, bb, nd);
                if (c.kind) {
                    Box kids[2];
                    const int nk = children(bb, c, kids);
                    double mn = 0.0;
                    for (int t = 0; t < nk; ++t) { const double e = tight_eff(M, kids[t]); mn = t == 0 ? e : std::min(mn, e); }
                    if (nk && mn > eff + 1e-12) {
                        for (int t = 0; t < nk; ++t) stack.push_back(kids[t]);
                        continue;
                    }
                }
            }
            if (!emit(bb, eff)) { *nboxes = -1; return ADJ_ERR_BAD_ARG; }
            continue;
        }
        Cut c;
        if (oversize && eff >= efficiency) {
            const int axis = argmax_shape(bb, nd);
            c = Cut{2, axis, (bb.hi[axis] - bb.lo[axis] + 1) / 2 - 1};
        } else {
            c = choose_cut(M, bb, nd);
        }
        if (!c.kind) {
            if (!emit(bb, eff)) { *nboxes = -1; return ADJ_ERR_BAD_ARG; }
            continue;
        }
        Box kids[2];
        const int nk = children(bb, c, kids);
        for (int t = 0; t < nk; ++t) stack.push_back(kids[t]);
    }
    *nboxes = n_out;
    return ADJ_OK;
}
