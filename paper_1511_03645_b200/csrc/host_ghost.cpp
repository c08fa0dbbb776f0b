// Host-native ghost-rectangle construction of one level (amr.build_ghost_rects:
// per patch ghost strip, the same-level COPY overlaps, then the COARSE pieces
// of what is left), same rectangles in the same order as the Python
// restatement.  The reference fills ghosts per patch (fill_ghost_same_level /
// fill_ghost_from_coarse, solver.py:208-263); these rectangles drive the
// batched K2 launches and the planned gather.
//
// Overlap queries use a uniform bin grid over the level index space instead
// of scanning every box, so a level of thousands of patches costs O(P).
#include <stdint.h>
#include <string.h>
#include <algorithm>
#include <vector>

#include "../../include/adjamr_b200.h"

namespace {

struct Box {
    int lo[2], hi[2];
};

bool intersect(const Box& a, const Box& b, int nd, Box& out) {
    for (int d = 0; d < nd; ++d) {
        out.lo[d] = std::max(a.lo[d], b.lo[d]);
        out.hi[d] = std::min(a.hi[d], b.hi[d]);
        if (out.lo[d] > out.hi[d]) return false;
    }
    if (nd == 1) { out.lo[1] = out.hi[1] = 0; }
    return true;
}

int64_t cells(const Box& b, int nd) {
    int64_t n = 1;
    for (int d = 0; d < nd; ++d) n *= (int64_t)(b.hi[d] - b.lo[d] + 1);
    return n;
}

// Boxes binned on a coarse grid; query returns overlapping indices ascending.
struct Index {
    int nd, bin, nbx, nby;
    const std::vector<Box>* boxes;
    std::vector<std::vector<int>> bins;
    std::vector<int> stamp;
    int tick = 0;
    void build(const std::vector<Box>& bx, int nd_, int extent_x, int extent_y) {
        boxes = &bx;
        nd = nd_;
        int64_t area = 0;
        for (const Box& b : bx) area += cells(b, nd);
        const double mean = bx.empty() ? 1.0 : (double)area / (double)bx.size();
        bin = std::max(8, (int)(nd == 2 ? __builtin_sqrt(mean) : mean));
        nbx = std::max(1, (extent_x + bin - 1) / bin + 2);
        nby = nd == 2 ? std::max(1, (extent_y + bin - 1) / bin + 2) : 1;
        bins.assign((size_t)nbx * nby, {});
        stamp.assign(bx.size(), -1);
        for (int k = 0; k < (int)bx.size(); ++k) {
            int x0, x1, y0, y1;
            range(bx[k], x0, x1, y0, y1);
            for (int i = x0; i <= x1; ++i)
                for (int j = y0; j <= y1; ++j) bins[(size_t)i * nby + j].push_back(k);
        }
    }
    void range(const Box& b, int& x0, int& x1, int& y0, int& y1) const {
        auto cl = [](int v, int n) { return v < 0 ? 0 : (v >= n ? n - 1 : v); };
        x0 = cl(b.lo[0] / bin + (b.lo[0] < 0 ? -1 : 0) + 1, nbx);
        x1 = cl(b.hi[0] / bin + (b.hi[0] < 0 ? -1 : 0) + 1, nbx);
        if (nd == 2) {
            y0 = cl(b.lo[1] / bin + (b.lo[1] < 0 ? -1 : 0) + 1, nby);
            y1 = cl(b.hi[1] / bin + (b.hi[1] < 0 ? -1 : 0) + 1, nby);
        } else {
            y0 = y1 = 0;
        }
    }
    void query(const Box& q, std::vector<int>& out) {
        out.clear();
        ++tick;
        int x0, x1, y0, y1;
        range(q, x0, x1, y0, y1);
        Box tmp;
        for (int i = x0; i <= x1; ++i)
            for (int j = y0; j <= y1; ++j)
                for (int k : bins[(size_t)i * nby + j]) {
                    if (stamp[k] == tick) continue;
                    stamp[k] = tick;
                    if (intersect((*boxes)[k], q, nd, tmp)) out.push_back(k);
                }
        std::sort(out.begin(), out.end());
    }
};

// _runs: maximal runs of true as (start, end) inclusive
void runs(const std::vector<uint8_t>& v, std::vector<std::pair<int, int>>& out) {
    out.clear();
    const int n = (int)v.size();
    int k = 0;
    while (k < n) {
        if (!v[k]) { ++k; continue; }
        int e = k;
        while (e + 1 < n && v[e + 1]) ++e;
        out.emplace_back(k, e);
        k = e + 1;
    }
}

// _subtract: cells of box not in any hole, as row runs along the longer axis
void subtract(const Box& box, const std::vector<Box>& holes, int nd, std::vector<Box>& out) {
    out.clear();
    const int sx = box.hi[0] - box.lo[0] + 1;
    const int sy = nd == 2 ? box.hi[1] - box.lo[1] + 1 : 1;
    std::vector<uint8_t> m((size_t)sx * sy, 1);
    Box ib;
    for (const Box& h : holes) {
        if (!intersect(box, h, nd, ib)) continue;
        for (int i = ib.lo[0]; i <= ib.hi[0]; ++i)
            for (int j = (nd == 2 ? ib.lo[1] : 0); j <= (nd == 2 ? ib.hi[1] : 0); ++j)
                m[(size_t)(i - box.lo[0]) * sy + (nd == 2 ? j - box.lo[1] : 0)] = 0;
    }
    bool all = true;
    for (uint8_t v : m) all = all && v;
    if (all) { out.push_back(box); return; }
    std::vector<uint8_t> line;
    std::vector<std::pair<int, int>> rr;
    if (nd == 1) {
        line.assign(m.begin(), m.end());
        runs(line, rr);
        for (auto& r : rr) { Box b{{box.lo[0] + r.first, 0}, {box.lo[0] + r.second, 0}}; out.push_back(b); }
        return;
    }
    if (sx <= sy) {
        for (int i = 0; i < sx; ++i) {
            line.assign(m.begin() + (size_t)i * sy, m.begin() + (size_t)(i + 1) * sy);
            runs(line, rr);
            for (auto& r : rr) out.push_back(Box{{box.lo[0] + i, box.lo[1] + r.first}, {box.lo[0] + i, box.lo[1] + r.second}});
        }
    } else {
        for (int j = 0; j < sy; ++j) {
            line.resize(sx);
            for (int i = 0; i < sx; ++i) line[i] = m[(size_t)i * sy + j];
            runs(line, rr);
            for (auto& r : rr) out.push_back(Box{{box.lo[0] + r.first, box.lo[1] + j}, {box.lo[0] + r.second, box.lo[1] + j}});
        }
    }
}

}  // namespace

extern "C" int adj_ghost_rects(int ndim, int ghost, const int32_t* level_shape, int npatch, const int32_t* lo,
                               const int32_t* hi, int ncoarse, const int32_t* clo, const int32_t* chi, int ratio,
                               int only, int disjoint, AdjRect* rects, int max_rects, int32_t* nrects,
                               int64_t* covered) {
    if ((ndim != 1 && ndim != 2) || ghost < 0 || !level_shape || npatch < 0 || (npatch && (!lo || !hi)) ||
        (ncoarse > 0 && (!clo || !chi || ratio < 1)) || !nrects || !covered || (max_rects > 0 && !rects))
        return ADJ_ERR_BAD_ARG;
    const int nd = ndim, g = ghost;
    std::vector<Box> same(npatch), cf(std::max(ncoarse, 0));
    for (int k = 0; k < npatch; ++k)
        for (int d = 0; d < 2; ++d) {
            same[k].lo[d] = d < nd ? lo[k * nd + d] : 0;
            same[k].hi[d] = d < nd ? hi[k * nd + d] : 0;
        }
    for (int c = 0; c < ncoarse; ++c)
        for (int d = 0; d < 2; ++d) {
            cf[c].lo[d] = d < nd ? clo[c * nd + d] * ratio : 0;
            cf[c].hi[d] = d < nd ? (chi[c * nd + d] + 1) * ratio - 1 : 0;
        }
    const int ex = level_shape[0], ey = nd == 2 ? level_shape[1] : 1;
    Index isame, icoarse;
    isame.build(same, nd, ex, ey);
    if (ncoarse > 0) icoarse.build(cf, nd, ex, ey);
    const Box dom{{0, 0}, {ex - 1, ey - 1}};
    int n = 0;
    bool overflow = false;
    auto emit = [&](int kind, int k, int src, const Box& ib, const Box* sbox) {
        if (n >= max_rects) { overflow = true; ++n; return; }
        AdjRect& r = rects[n++];
        memset(&r, 0, sizeof(r));
        r.kind = kind;
        r.dst_patch = k;
        r.src_patch = src;
        r.di0 = ib.lo[0] - (same[k].lo[0] - g);
        r.ni = ib.hi[0] - ib.lo[0] + 1;
        if (nd == 2) {
            r.dj0 = ib.lo[1] - (same[k].lo[1] - g);
            r.nj = ib.hi[1] - ib.lo[1] + 1;
        } else {
            r.nj = 1;
        }
        if (sbox) {
            r.si0 = ib.lo[0] - (sbox->lo[0] - g);
            if (nd == 2) r.sj0 = ib.lo[1] - (sbox->lo[1] - g);
        }
    };
    std::vector<int> cand;
    std::vector<Box> holes, pieces;
    for (int k = 0; k < npatch; ++k) {
        covered[k] = 0;
        if (only >= 0 && k != only) continue;
        const Box& p = same[k];
        Box strips[4];
        int ns;
        if (nd == 1) {
            strips[0] = Box{{p.lo[0] - g, 0}, {p.lo[0] - 1, 0}};
            strips[1] = Box{{p.hi[0] + 1, 0}, {p.hi[0] + g, 0}};
            ns = 2;
        } else {
            strips[0] = Box{{p.lo[0] - g, p.lo[1] - g}, {p.lo[0] - 1, p.hi[1] + g}};
            strips[1] = Box{{p.hi[0] + 1, p.lo[1] - g}, {p.hi[0] + g, p.hi[1] + g}};
            strips[2] = Box{{p.lo[0], p.lo[1] - g}, {p.hi[0], p.lo[1] - 1}};
            strips[3] = Box{{p.lo[0], p.hi[1] + 1}, {p.hi[0], p.hi[1] + g}};
            ns = 4;
        }
        for (int s = 0; s < ns; ++s) {
            Box box;
            if (!intersect(strips[s], dom, nd, box)) continue;
            holes.clear();
            isame.query(box, cand);
            for (int o : cand) {
                if (o == k) continue;
                Box ib;
                if (!intersect(box, same[o], nd, ib)) continue;
                emit(ADJ_RECT_COPY, k, o, ib, &same[o]);
                holes.push_back(ib);
                covered[k] += cells(ib, nd);
            }
            if (ncoarse > 0) {
                if (disjoint) subtract(box, holes, nd, pieces);
                else { pieces.clear(); pieces.push_back(box); }
                for (const Box& piece : pieces) {
                    icoarse.query(piece, cand);
                    for (int c : cand) {
                        Box ib;
                        if (!intersect(piece, cf[c], nd, ib)) continue;
                        emit(ADJ_RECT_COARSE, k, c, ib, nullptr);
                        if (disjoint) covered[k] += cells(ib, nd);
                    }
                }
                if (!disjoint) {
                    icoarse.query(box, cand);
                    for (int c : cand) {
                        Box ib;
                        if (intersect(box, cf[c], nd, ib)) covered[k] += cells(ib, nd);
                    }
                    for (const Box& h : holes) covered[k] -= cells(h, nd);
                }
            }
        }
    }
    *nrects = n;
    return overflow ? ADJ_ERR_BAD_ARG : ADJ_OK;
}

// Pairwise overlaps of dst boxes with (optionally refined) src boxes, as
// rectangles in dst ghost-inclusive coordinates (COPY: also src
// coordinates) -- the regrid fill of a new level from its parents (COARSE,
// src boxes refined by `ratio`) and from the old level (COPY),
// amr.py:504-551.  Order: dst ascending, then src ascending.
extern "C" int adj_box_overlaps(int ndim, int kind, int ndst, const int32_t* dlo, const int32_t* dhi, int gdst,
                                int nsrc, const int32_t* slo, const int32_t* shi, int gsrc, int ratio,
                                AdjRect* rects, int max_rects, int32_t* nrects) {
    if ((ndim != 1 && ndim != 2) || ndst < 0 || nsrc < 0 || ratio < 1 || !nrects || (max_rects > 0 && !rects) ||
        (ndst && (!dlo || !dhi)) || (nsrc && (!slo || !shi)))
        return ADJ_ERR_BAD_ARG;
    const int nd = ndim;
    std::vector<Box> dst(ndst), src(nsrc), orig(nsrc);
    int ex = 1, ey = 1;
    for (int k = 0; k < ndst; ++k)
        for (int d = 0; d < 2; ++d) {
            dst[k].lo[d] = d < nd ? dlo[k * nd + d] : 0;
            dst[k].hi[d] = d < nd ? dhi[k * nd + d] : 0;
        }
    for (int c = 0; c < nsrc; ++c)
        for (int d = 0; d < 2; ++d) {
            orig[c].lo[d] = d < nd ? slo[c * nd + d] : 0;
            orig[c].hi[d] = d < nd ? shi[c * nd + d] : 0;
            src[c].lo[d] = d < nd ? orig[c].lo[d] * ratio : 0;
            src[c].hi[d] = d < nd ? (orig[c].hi[d] + 1) * ratio - 1 : 0;
            ex = std::max(ex, src[c].hi[0] + 1);
            if (nd == 2) ey = std::max(ey, src[c].hi[1] + 1);
        }
    for (const Box& b : dst) { ex = std::max(ex, b.hi[0] + 1); if (nd == 2) ey = std::max(ey, b.hi[1] + 1); }
    Index idx;
    idx.build(src, nd, ex, ey);
    std::vector<int> cand;
    int n = 0;
    bool overflow = false;
    for (int k = 0; k < ndst; ++k) {
        idx.query(dst[k], cand);
        for (int c : cand) {
            Box ib;
            if (!intersect(dst[k], src[c], nd, ib)) continue;
            if (n >= max_rects) { overflow = true; ++n; continue; }
            AdjRect& r = rects[n++];
            memset(&r, 0, sizeof(r));
            r.kind = kind;
            r.dst_patch = k;
            r.src_patch = c;
            r.di0 = ib.lo[0] - (dst[k].lo[0] - gdst);
            r.ni = ib.hi[0] - ib.lo[0] + 1;
            r.nj = nd == 2 ? ib.hi[1] - ib.lo[1] + 1 : 1;
            if (nd == 2) r.dj0 = ib.lo[1] - (dst[k].lo[1] - gdst);
            if (kind == ADJ_RECT_COPY) {
                r.si0 = ib.lo[0] - (orig[c].lo[0] - gsrc);
                if (nd == 2) r.sj0 = ib.lo[1] - (orig[c].lo[1] - gsrc);
            }
        }
    }
    *nrects = n;
    return overflow ? ADJ_ERR_BAD_ARG : ADJ_OK;
}
