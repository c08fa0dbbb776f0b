"""Multilevel driver: device level sweep + host clustering and bookkeeping.

Drop-in for the reference's amr.py (/root/reference/pkg/src/adjamr/amr.py).
The level sweep is device work: ghost fill (K2: coarse space-time
interpolation, same-level copies, physical boundaries -- amr.py:479-491),
the batched patch step (K1), fine-to-coarse averaging (K4, amr.py:399-450),
adjoint flagging of a whole level in one K3 launch, and the regrid data
movement (new interiors from the parent and old patches, amr.py:504-551).
Flag buffering, signature-bisection clustering, nesting clip and patch
bookkeeping stay on the host, as north_star prescribes.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib, device
from .geometry import Patch, PatchHierarchy, allowed_region_mask
from .solver import (BoundarySpec, CflViolationError, NumericalBlowupError, SchedulingError,
                     level_store, sample_patch_material)


@dataclass
class FlagField:
    flags: np.ndarray
    lo: tuple[int, ...]
    level: int
    strategy_name: str
    time: float


@dataclass(frozen=True)
class ClusterBox:
    lo: tuple[int, ...]
    hi: tuple[int, ...]
    efficiency: float

    @property
    def shape(self):
        return tuple(h - l + 1 for l, h in zip(self.lo, self.hi))


@dataclass(frozen=True)
class RefinementRegion:
    min_level: int
    max_level: int
    t1: float
    t2: float
    rect: tuple[float, ...]

    def __post_init__(self):
        if self.min_level > self.max_level:
            raise ValueError("min_level must be <= max_level")

    def contains_time(self, t: float) -> bool:
        return self.t1 <= t <= self.t2

    def cell_mask(self, spec) -> np.ndarray:
        cs = spec.cell_centers()
        inx = (cs[0] >= self.rect[0]) & (cs[0] <= self.rect[1])
        if spec.ndim == 1:
            return inx
        iny = (cs[1] >= self.rect[2]) & (cs[1] <= self.rect[3])
        return np.logical_and.outer(inx, iny)


# ---------------------------------------------------------------------------
# flagging strategies (amr.py:75-134); the adjoint one lives in adjoint.py


class FlaggingStrategy:
    name = "base"

    def evaluate(self, patch: Patch) -> np.ndarray:
        raise NotImplementedError


class DifferenceFlagging(FlaggingStrategy):
    name = "difference"

    def __init__(self, tolerance: float):
        if tolerance <= 0:
            raise ValueError("tolerance must be positive")
        self.tolerance = tolerance

    def evaluate(self, patch):
        g = patch.spec.ghost_width
        q = patch.state
        shape = patch.spec.shape
        big = np.zeros(shape)
        for axis in range(patch.spec.ndim):
            d = np.abs(np.diff(q, axis=1 + axis))
            for start in (g - 1, g):
                sl = [slice(g, g + n) for n in shape]
                sl[axis] = slice(start, start + shape[axis])
                big = np.maximum(big, np.max(d[(slice(None), *sl)], axis=0))
        return big > self.tolerance


class SurfaceFlagging(FlaggingStrategy):
    name = "surface"

    def __init__(self, tolerance: float):
        if tolerance <= 0:
            raise ValueError("tolerance must be positive")
        self.tolerance = tolerance

    def evaluate(self, patch):
        sl = patch.spec.interior_slices()
        flags = np.abs(patch.state[(0, *sl)]) > self.tolerance
        if hasattr(patch.aux, "wet"):
            flags &= patch.aux.wet[sl]
        return flags


class EverywhereFlagging(FlaggingStrategy):
    name = "everywhere"

    def evaluate(self, patch):
        return np.ones(patch.spec.shape, dtype=bool)


def _apply_regions(flags, spec, t, regions):
    new_level = spec.level + 1
    for r in regions:
        if r.contains_time(t) and new_level <= r.min_level:
            flags |= r.cell_mask(spec)
    for r in regions:
        if r.contains_time(t) and new_level > r.max_level:
            flags &= ~r.cell_mask(spec)
    return flags


def flag_cells(patch: Patch, strategy: FlaggingStrategy, regions=()) -> FlagField:
    """Strategy flags then region overrides (amr.py:137-154)."""
    flags = np.array(strategy.evaluate(patch), dtype=bool)
    flags = _apply_regions(flags, patch.spec, patch.time, regions)
    return FlagField(flags=flags, lo=patch.spec.lo, level=patch.spec.level,
                     strategy_name=strategy.name, time=patch.time)


def buffer_flags(flags: FlagField, buffer_cells: int) -> FlagField:
    """Box dilation of radius buffer_cells, clipped to the patch (amr.py:157-179)."""
    if buffer_cells < 0:
        raise ValueError("buffer_cells must be >= 0")
    out = flags.flags.copy()
    for axis in range(out.ndim):
        grown = out.copy()
        n = out.shape[axis]
        for s in range(1, min(buffer_cells, n - 1) + 1):
            a = [slice(None)] * out.ndim
            b = [slice(None)] * out.ndim
            a[axis], b[axis] = slice(0, n - s), slice(s, n)
            grown[tuple(a)] |= out[tuple(b)]
            grown[tuple(b)] |= out[tuple(a)]
        out = grown
    return FlagField(flags=out, lo=flags.lo, level=flags.level, strategy_name=flags.strategy_name,
                     time=flags.time)


# ---------------------------------------------------------------------------
# signature-bisection clustering (amr.py:186-337)


def _sig(mask, axis):
    other = tuple(a for a in range(mask.ndim) if a != axis)
    return mask.sum(axis=other) if other else mask.astype(int)


def _bbox(mask):
    nz = np.nonzero(mask)
    if nz[0].size == 0:
        return None
    return tuple(int(a.min()) for a in nz), tuple(int(a.max()) for a in nz)


def _choose_cut(sub):
    """Hole nearest the centre (best over axes), else the strongest Laplacian
    sign change of the signature, else the midpoint of the longest axis."""
    best = None
    for axis in range(sub.ndim):
        sig = _sig(sub, axis)
        holes = np.flatnonzero(sig == 0)
        if holes.size:
            mid = (sig.size - 1) / 2.0
            k = int(holes[np.argmin(np.abs(holes - mid))])
            score = abs(k - mid) / max(sig.size, 1)
            if best is None or score < best[0]:
                best = (score, axis, k)
    if best is not None:
        return "hole", best[1], best[2]
    best = None
    for axis in range(sub.ndim):
        sig = _sig(sub, axis)
        n = sig.size
        if n < 4:
            continue
        lap = sig[2:] - 2 * sig[1:-1] + sig[:-2]
        mid = (n - 1) / 2.0
        for k in range(lap.size - 1):
            if lap[k] * lap[k + 1] < 0:
                key = (abs(lap[k + 1] - lap[k]), -abs((k + 1.5) - mid))
                if best is None or key > best[0]:
                    best = (key, axis, k + 1)
    if best is not None:
        return "edge", best[1], best[2]
    axis = int(np.argmax(sub.shape))
    if sub.shape[axis] < 2:
        return None
    return "edge", axis, sub.shape[axis] // 2 - 1


def _children(lo, hi, cut):
    kind, axis, k = cut
    a_hi, b_lo = list(hi), list(lo)
    if kind == "hole":
        a_hi[axis] = lo[axis] + k - 1
        b_lo[axis] = lo[axis] + k + 1
    else:
        a_hi[axis] = lo[axis] + k
        b_lo[axis] = lo[axis] + k + 1
    kids = []
    if a_hi[axis] >= lo[axis]:
        kids.append((tuple(lo), tuple(a_hi)))
    if hi[axis] >= b_lo[axis]:
        kids.append((tuple(b_lo), tuple(hi)))
    return kids


def _box_slice(lo, hi):
    return tuple(slice(l, h + 1) for l, h in zip(lo, hi))


def _tight_efficiency(mask, box):
    sub = mask[_box_slice(*box)]
    bb = _bbox(sub)
    if bb is None:
        return 1.0
    core = sub[_box_slice(*bb)]
    return float(core.sum()) / core.size


def cluster(flags, efficiency_threshold: float, max_edge: int | None = None,
            native: bool | None = None) -> list[ClusterBox]:
    """Cover all flagged cells with efficient rectangles (amr.py:244-309).

    Runs the host-native C++ port (``adj_cluster`` in libadjamr_b200.so,
    O(perimeter) per candidate box via prefix sums) when the library is
    built, else the same algorithm in numpy; both produce identical boxes."""
    if not 0.0 < efficiency_threshold <= 1.0:
        raise ValueError("efficiency_threshold must be in (0, 1]")
    if isinstance(flags, FlagField):
        mask, offset = flags.flags, flags.lo
    else:
        mask = np.asarray(flags, dtype=bool)
        offset = (0,) * mask.ndim
    if native is not False:
        # the algorithm starts from the flags' bounding box (amr.py:258-262):
        # clustering the cropped mask gives the same boxes
        nz = [np.flatnonzero(mask.any(axis=tuple(b for b in range(mask.ndim) if b != a)))
              for a in range(mask.ndim)]
        if any(len(v) == 0 for v in nz):
            return []
        crop = tuple(slice(int(v[0]), int(v[-1]) + 1) for v in nz)
        mask = mask[crop]
        offset = tuple(o + int(v[0]) for o, v in zip(offset, nz))
        out = _cluster_native(mask, offset, efficiency_threshold, max_edge)
        if out is not None:
            return out
        if native:
            raise RuntimeError("native clustering unavailable")
    return _cluster_py(mask, offset, efficiency_threshold, max_edge)


def _cluster_native(mask, offset, eff, max_edge):
    try:
        lib = _lib.load_library()
    except _lib.NativeUnavailableError:
        return None
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    nd = m.ndim
    nx, ny = m.shape[0], (m.shape[1] if nd == 2 else 1)
    cap = max(16, int(m.sum()) + 1)
    boxes = np.zeros((cap, 4), dtype=np.int32)
    effs = np.zeros(cap, dtype=np.float64)
    n = _lib.I32()
    rc = lib.adj_cluster(m.ctypes.data, nd, nx, ny, float(eff), -1 if max_edge is None else int(max_edge),
                         boxes.ctypes.data, effs.ctypes.data, cap, _lib.C.byref(n))
    _lib.check(rc, "adj_cluster")
    out = []
    for k in range(n.value):
        b = boxes[k]
        lo = (int(b[0]) + offset[0],) if nd == 1 else (int(b[0]) + offset[0], int(b[1]) + offset[1])
        hi = (int(b[2]) + offset[0],) if nd == 1 else (int(b[2]) + offset[0], int(b[3]) + offset[1])
        out.append(ClusterBox(lo=lo, hi=hi, efficiency=float(effs[k])))
    return out


def _cluster_py(mask, offset, efficiency_threshold, max_edge):
    boxes: list[ClusterBox] = []
    top = _bbox(mask)
    if top is None:
        return boxes
    todo = [top]

    def emit(lo, hi, eff):
        boxes.append(ClusterBox(lo=tuple(l + o for l, o in zip(lo, offset)),
                                hi=tuple(h + o for h, o in zip(hi, offset)), efficiency=eff))

    while todo:
        lo, hi = todo.pop()
        bb = _bbox(mask[_box_slice(lo, hi)])
        if bb is None:
            continue
        lo, hi = tuple(l + b for l, b in zip(lo, bb[0])), tuple(l + b for l, b in zip(lo, bb[1]))
        sub = mask[_box_slice(lo, hi)]
        eff = int(sub.sum()) / sub.size
        oversize = max_edge is not None and max(sub.shape) > max_edge
        if eff >= efficiency_threshold and not oversize:
            if eff < 1.0:
                cut = _choose_cut(sub)
                if cut is not None:
                    kids = _children(lo, hi, cut)
                    effs = [_tight_efficiency(mask, kb) for kb in kids]
                    if effs and min(effs) > eff + 1e-12:
                        todo.extend(kids)
                        continue
            emit(lo, hi, eff)
            continue
        if oversize and eff >= efficiency_threshold:
            axis = int(np.argmax(sub.shape))
            cut = ("edge", axis, sub.shape[axis] // 2 - 1)
        else:
            cut = _choose_cut(sub)
        if cut is None:
            emit(lo, hi, eff)
            continue
        todo.extend(_children(lo, hi, cut))
    return boxes


def _runs(row):
    """Maximal runs of True as (start, end) inclusive."""
    v = np.concatenate([[False], np.asarray(row, dtype=bool), [False]])
    d = np.diff(v.astype(np.int8))
    starts = np.flatnonzero(d == 1)
    ends = np.flatnonzero(d == -1) - 1
    return [(int(a), int(b)) for a, b in zip(starts, ends)]


def _allowed_rectangles(box: ClusterBox, allowed, mask):
    """Trim a box to the nesting-allowed region (amr.py:344-382)."""
    sub = allowed[_box_slice(box.lo, box.hi)]
    if sub.all():
        return [box]
    rects = []
    if sub.ndim == 1:
        rects = [((box.lo[0] + a,), (box.lo[0] + b,)) for a, b in _runs(sub)]
    else:
        i = 0
        while i < sub.shape[0]:
            runs = _runs(sub[i])
            j = i
            while j + 1 < sub.shape[0] and _runs(sub[j + 1]) == runs:
                j += 1
            rects += [((box.lo[0] + i, box.lo[1] + a), (box.lo[0] + j, box.lo[1] + b)) for a, b in runs]
            i = j + 1
    out = []
    for lo, hi in rects:
        f = mask[_box_slice(lo, hi)]
        if f.any():
            out.append(ClusterBox(lo=lo, hi=hi, efficiency=int(f.sum()) / f.size))
    return out


# ---------------------------------------------------------------------------
# context


@dataclass
class AmrContext:
    equation: object
    boundary: BoundarySpec
    strategy: FlaggingStrategy
    limiter: str = "MC"
    regions: tuple = ()
    regrid_interval: int = 1
    buffer_cells: int = 3
    efficiency: float = 0.7
    max_patch_edge: int = 60
    step_counts: dict = field(default_factory=dict)
    cell_steps: dict = field(default_factory=dict)
    flagged_per_regrid: list = field(default_factory=list)
    on_level_advanced: object = None
    variant: int = _lib.VARIANT_FAST

    def count_step(self, level: int, cells: int):
        self.cell_steps[level] = self.cell_steps.get(level, 0) + cells


# ---------------------------------------------------------------------------
# device ghost fill (K2) with host-built rectangle lists


def _ghost_strips(spec):
    """Ghost ring of a patch as global-index boxes (lo, hi) inclusive."""
    g = spec.ghost_width
    if spec.ndim == 1:
        return [((spec.lo[0] - g,), (spec.lo[0] - 1,)), ((spec.hi[0] + 1,), (spec.hi[0] + g,))]
    (x0, y0), (x1, y1) = spec.lo, spec.hi
    return [((x0 - g, y0 - g), (x0 - 1, y1 + g)), ((x1 + 1, y0 - g), (x1 + g, y1 + g)),
            ((x0, y0 - g), (x1, y0 - 1)), ((x0, y1 + 1), (x1, y1 + g))]


def _intersect(alo, ahi, blo, bhi):
    lo = tuple(max(a, b) for a, b in zip(alo, blo))
    hi = tuple(min(a, b) for a, b in zip(ahi, bhi))
    return None if any(l > h for l, h in zip(lo, hi)) else (lo, hi)


def _boxes(patches):
    lo = np.array([p.spec.lo for p in patches], dtype=np.int64)
    hi = np.array([p.spec.hi for p in patches], dtype=np.int64)
    return lo, hi


def _candidates(lo_arr, hi_arr, qlo, qhi):
    ok = np.ones(len(lo_arr), dtype=bool)
    for a in range(lo_arr.shape[1]):
        ok &= (lo_arr[:, a] <= qhi[a]) & (hi_arr[:, a] >= qlo[a])
    return np.flatnonzero(ok)


def _rect(kind, dst, src, dlo, dspec, extent, slo=None, sspec=None):
    g = dspec.ghost_width
    di = [dlo[a] - (dspec.lo[a] - g) for a in range(dspec.ndim)]
    si = [0, 0]
    if slo is not None:
        gs = sspec.ghost_width
        si = [slo[a] - (sspec.lo[a] - gs) for a in range(sspec.ndim)]
    if dspec.ndim == 1:
        return (kind, dst, src, di[0], 0, extent[0], 1, si[0], 0, 0)
    return (kind, dst, src, di[0], di[1], extent[0], extent[1], si[0], si[1], 0)


def _subtract(box, holes):
    """Cells of ``box`` (lo, hi) not in any of ``holes``, as rectangles
    (row runs along the box's longer axis; ghost strips are 2 cells thick)."""
    (lo, hi) = box
    shape = tuple(h - l + 1 for l, h in zip(lo, hi))
    m = np.ones(shape, dtype=bool)
    for hl, hh in holes:
        ib = _intersect(lo, hi, hl, hh)
        if ib is not None:
            m[tuple(slice(a - l, b - l + 1) for a, b, l in zip(ib[0], ib[1], lo))] = False
    if m.all():
        return [box]
    out = []
    if m.ndim == 1:
        for a, b in _runs(m):
            out.append(((lo[0] + a,), (lo[0] + b,)))
        return out
    if shape[0] <= shape[1]:
        for i in range(shape[0]):
            for a, b in _runs(m[i]):
                out.append(((lo[0] + i, lo[1] + a), (lo[0] + i, lo[1] + b)))
    else:
        for j in range(shape[1]):
            for a, b in _runs(m[:, j]):
                out.append(((lo[0] + a, lo[1] + j), (lo[0] + b, lo[1] + j)))
    return out


def build_ghost_rects(hierarchy: PatchHierarchy, level: int, only=None, disjoint: bool = False, native=None):
    """Rectangles for the in-domain ghost phases of one level:
    coarse rects grouped by coarse patch, then same-level copy rects.
    ``disjoint``: coarse rects exclude the cells a same-level copy overwrites
    (same final values, one launch, less interpolation).
    Returns (coarse {coarse slot: [rect]}, copy [rect], covered cells per patch).
    Runs natively (adj_ghost_rects) when the library is present."""
    if native is not False:
        try:
            return _build_ghost_rects_native(hierarchy, level, only, disjoint)
        except _lib.NativeUnavailableError:
            if native:
                raise
    return _build_ghost_rects_py(hierarchy, level, only, disjoint)


def _build_ghost_rects_native(hierarchy, level, only, disjoint):
    import ctypes as C
    patches = hierarchy.patches(level)
    nd = hierarchy.ndim
    shape = np.array(hierarchy.level_shape(level), dtype=np.int32)
    lo, hi = (np.ascontiguousarray(a, dtype=np.int32) for a in _boxes(patches))
    coarse = hierarchy.patches(level - 1) if level >= 2 else []
    if coarse:
        clo, chi = (np.ascontiguousarray(a, dtype=np.int32) for a in _boxes(coarse))
        r = hierarchy.ratio_to_finer(level - 1)
    else:
        clo = chi = np.zeros((1, nd), np.int32)
        r = 1
    k_only = -1 if only is None else next(k for k, p in enumerate(patches) if p is only)
    g = patches[0].spec.ghost_width
    cap = max(64, 16 * len(patches))
    lib = _lib.load_library()
    while True:
        rects = np.zeros(cap, dtype=_lib.RECT_DTYPE)
        covered = np.zeros(len(patches), dtype=np.int64)
        n = _lib.I32()
        rc = lib.adj_ghost_rects(nd, g, shape.ctypes.data, len(patches), lo.ctypes.data, hi.ctypes.data,
                                 len(coarse), clo.ctypes.data, chi.ctypes.data, r, k_only, int(disjoint),
                                 rects.ctypes.data, cap, C.byref(n), covered.ctypes.data)
        if rc == 0:
            break
        if n.value <= cap:
            raise ValueError("adj_ghost_rects: bad arguments")
        cap = n.value
    rects = rects[: n.value]
    copy_rects = rects[rects["kind"] == _lib.RECT_COPY].tolist()
    coarse_rects: dict[int, list] = {}
    for r_ in rects[rects["kind"] == _lib.RECT_COARSE].tolist():
        coarse_rects.setdefault(r_[2], []).append(r_)
    return coarse_rects, copy_rects, covered


def _build_ghost_rects_py(hierarchy: PatchHierarchy, level: int, only=None, disjoint: bool = False):
    patches = hierarchy.patches(level)
    shape = hierarchy.level_shape(level)
    dom_lo, dom_hi = (0,) * hierarchy.ndim, tuple(n - 1 for n in shape)
    same_lo, same_hi = _boxes(patches)
    coarse = hierarchy.patches(level - 1) if level >= 2 else []
    r = hierarchy.ratio_to_finer(level - 1) if level >= 2 else 1
    if coarse:
        c_lo, c_hi = _boxes(coarse)
        cf_lo, cf_hi = c_lo * r, (c_hi + 1) * r - 1
    coarse_rects: dict[int, list] = {}
    copy_rects = []
    covered = np.zeros(len(patches), dtype=np.int64)
    for k, p in enumerate(patches):
        if only is not None and p is not only:
            continue
        for slo, shi in _ghost_strips(p.spec):
            box = _intersect(slo, shi, dom_lo, dom_hi)
            if box is None:
                continue
            # physical cells of this strip are out of domain; in-domain part only
            holes = []
            for o in _candidates(same_lo, same_hi, *box):
                if o == k:
                    continue
                ib = _intersect(*box, tuple(same_lo[o]), tuple(same_hi[o]))
                if ib is not None:
                    ext = [h - l + 1 for l, h in zip(*ib)]
                    copy_rects.append(_rect(_lib.RECT_COPY, k, int(o), ib[0], p.spec, ext, ib[0],
                                            patches[o].spec))
                    holes.append(ib)
                    covered[k] += int(np.prod(ext))
            if coarse:
                pieces = _subtract(box, holes) if disjoint else [box]
                for piece in pieces:
                    for c in _candidates(cf_lo, cf_hi, *piece):
                        ib = _intersect(*piece, tuple(cf_lo[c]), tuple(cf_hi[c]))
                        if ib is not None:
                            ext = [h - l + 1 for l, h in zip(*ib)]
                            coarse_rects.setdefault(int(c), []).append(
                                _rect(_lib.RECT_COARSE, k, int(c), ib[0], p.spec, ext))
                            if disjoint:
                                covered[k] += int(np.prod(ext))
                if not disjoint:
                    # coverage of the strip by coarse interpolation alone
                    for c in _candidates(cf_lo, cf_hi, *box):
                        ib = _intersect(*box, tuple(cf_lo[c]), tuple(cf_hi[c]))
                        if ib is not None:
                            covered[k] += int(np.prod([h - l + 1 for l, h in zip(*ib)]))
                    covered[k] -= sum(int(np.prod([h - l + 1 for l, h in zip(*hb)])) for hb in holes)
    return coarse_rects, copy_rects, covered


def _ring_and_physical(spec, level_shape):
    """(ghost ring size, out-of-domain ghost cells) of a patch."""
    g = spec.ghost_width
    tot = np.prod([n + 2 * g for n in spec.shape]) - np.prod(spec.shape)
    ind = 1
    for a in range(spec.ndim):
        lo = max(spec.lo[a] - g, 0)
        hi = min(spec.hi[a] + g, level_shape[a] - 1)
        ind *= hi - lo + 1
    return int(tot), int(np.prod([n + 2 * g for n in spec.shape]) - ind)


def _ring_and_physical_all(patches, level_shape):
    """_ring_and_physical of every patch, vectorised -> (ring, physical) arrays."""
    lo, hi = _boxes(patches)
    g = patches[0].spec.ghost_width
    n = hi - lo + 1
    full = np.prod(n + 2 * g, axis=1)
    ind = np.prod(np.minimum(hi + g, np.array(level_shape) - 1) - np.maximum(lo - g, 0) + 1, axis=1)
    return full - np.prod(n, axis=1), full - ind


# FAST sweeps: a coarse time weight below this is taken as 0 (old state only).  At the first
# substep of an interval t equals the coarse level's saved time up to the rounding drift of the
# subcycled level clocks (w ~ 1e-16 .. 1e-13 over C5's run); the reference then blends in
# w * q(t1), a change of at most w * |q(t1) - q(t0)| to the ghost value, far inside the FAST
# tolerance.  With w exactly 0 the first substep provably reads only the saved state, which
# lets a captured sweep overlap the coarse level's step with it (USE_LEVEL_OVERLAP).  The EXACT
# variant keeps the reference's blend bitwise.
SNAP_W = 1e-12


def _coarse_time_mode(cp: Patch, t: float, snap: bool = False):
    """space_time_interp scheduling (solver.py:266-286) -> (mode, w)."""
    eps = 1e-9 * max(abs(cp.time), 1.0)
    has_old = cp.time_old is not None and (
        (cp._store is not None and cp._store.has_old(cp._slot)) or cp._host_old is not None)
    if not has_old:
        if abs(t - cp.time) > eps:
            raise SchedulingError(f"coarse patch has no saved state bracketing t={t} (at {cp.time})")
        return 2, 1.0
    t0, t1 = cp.time_old, cp.time
    if not t0 - eps <= t <= t1 + eps:
        raise SchedulingError(f"t={t} outside coarse bracket [{t0}, {t1}]")
    if t1 == t0:
        return 0, 0.0
    w = float(np.clip((t - t0) / (t1 - t0), 0.0, 1.0))
    if w == 0.0 or (snap and w < SNAP_W):
        return 0, 0.0
    return 1, w


def _coarse_old_buffer(cst):
    """Device buffer holding every coarse patch's state_old (uploading host
    copies for patches whose saved state only exists on the host)."""
    import torch
    if cst.old is not None and bool(np.all(cst.old_valid)):
        return cst.buf[cst.old]
    need = [p for p in cst.patches if not cst.has_old(p._slot) and p._host_old is not None]
    if need:
        if cst.old is None or cst.old == cst.cur:
            if cst.old == cst.cur:
                cst._unalias()
            cst.old = cst._free(cst.cur, cst.ghost_src)
        for p in need:
            cst.view(p._slot, "old").copy_(torch.from_numpy(p._host_old))
            cst.old_valid[p._slot] = True
            p._host_old = None
    return cst.buf[cst.old] if cst.old is not None else cst.buf[cst.cur]


def fill_from_coarse(hierarchy: PatchHierarchy, level: int, t: float, only=None, _rects=None):
    """In-domain ghosts of one level (or of the patch ``only``) by coarse
    space-time interpolation (solver.py:227-286)."""
    patches = hierarchy.patches(level)
    coarse = hierarchy.patches(level - 1)
    if level < 2 or not patches or not coarse:
        return
    st = level_store(patches)
    cst = level_store(coarse)
    st.sync_in()
    cst.sync_in()
    cst.fold_ghosts()
    crects, _, _ = _rects if _rects is not None else build_ghost_rects(hierarchy, level, only)
    if not crects:
        return
    st.prepare_write(full_ghosts=False)
    old_buf = _coarse_old_buffer(cst)
    groups: dict = {}
    for c, rl in crects.items():
        groups.setdefault(_coarse_time_mode(coarse[c], t), []).extend(rl)
    r = hierarchy.ratio_to_finer(level - 1)
    for (mode, w), rl in groups.items():
        device.coarse_rects(st, cst, np.array(rl, dtype=_lib.RECT_DTYPE), old_buf, cst.buf[cst.cur],
                            hierarchy, r, w, mode)


def fill_same_level(level_patches, only=None, _rects=None):
    if not level_patches:
        return
    st = level_store(level_patches)
    st.sync_in()
    if _rects is None:
        h = _pseudo_hierarchy(level_patches)
        _, rects, _ = build_ghost_rects(h, 1, only)
    else:
        rects = _rects
    if not rects:
        return
    st.prepare_write(full_ghosts=False)
    device.copy_rects(st, st, np.array(rects, dtype=_lib.RECT_DTYPE), st.buf[st.cur], st.buf[st.cur])


def _pseudo_hierarchy(patches):
    """A one-level hierarchy wide enough to hold the patches (same-level rects only)."""
    hi = np.max([p.spec.hi for p in patches], axis=0) + 1 + patches[0].spec.ghost_width
    nd = patches[0].spec.ndim
    h = PatchHierarchy(xlim=(0.0, 1.0), ylim=None if nd == 1 else (0.0, 1.0),
                       base_shape=tuple(int(v) for v in hi), ratios=[])
    h.levels = [list(patches)]
    return h


def _fill_physical_subset(st, slots, boundary, equation, level_shape):
    device.fill_physical(st, boundary, equation, level_shape, slots=slots)


# planned whole-level ghost fill (device.GhostPlan); False: the three-phase launches
USE_GHOST_PLAN = True
# planned restriction (device.RestrictPlan, one thread per coarse cell); False: per-rect blocks
USE_RESTRICT_PLAN = True
# finest level's last substep on the fast static-CFL path: restriction into the coarser level
# fused into the step launch (device.FusedRestrict); False: a separate K4 launch
USE_FUSED_RESTRICT = True
# fast static-CFL levels: run the planned fill inside the step launch (prefill + grid barrier).
# Off: measured slower on C5 (0.94-0.96 vs 0.75 ms per coarse step) -- the persistent step grid
# has ~57K threads for ~400K gather entries, the standalone gather ~300K
USE_FUSED_FILL = False
# fast static-CFL levels of small patches: the level's fill runs per warp job inside the step
# launch (device.JobFill; no grid barrier, no separate gather launch); coarse-interpolated ghost
# values of a coarse interval are computed in its first substep and reused from a cache after.
# Opt-in (ADJAMR_JOB_FILL=1): measured on C5 0.93 vs 0.76 ms per coarse step -- a cached-substep
# launch costs what the separate gather + step did (51.9 vs 51.3 us on L3), a first substep
# (coarse values at both times) far more (93.5 vs 54.8 us): every warp fills before it marches
USE_JOB_FILL = os.environ.get("ADJAMR_JOB_FILL", "0") == "1"


def _static_fast(st, ctx) -> bool:
    return ctx.variant == _lib.VARIANT_FAST and st.ndim == 2 and not st.any_dry() and not st.two_rows()


class LevelPlan:
    """Launch plan of one level for the batched sweep: its store, the coarse
    store, device-resident ghost / restriction rectangle tables and the
    coverage flag.  Rebuilt only when the level's patch list changes (regrid)."""

    def __init__(self, hierarchy: PatchHierarchy, level: int):
        patches = hierarchy.patches(level)
        self.plist = hierarchy.levels[level - 1]
        self.n = len(patches)
        self.ends = (patches[0], patches[-1])
        self.st = level_store(patches)
        self.clist = hierarchy.levels[level - 2] if level >= 2 else None
        coarse = hierarchy.patches(level - 1) if level >= 2 else []
        self.cst = level_store(coarse) if coarse else None
        crects, copies, covered = build_ghost_rects(hierarchy, level)
        self.crects_by_patch = crects            # full strips (unsynchronised fallback)
        self.copies = device.RectTable(copies)
        dcr, _, _ = build_ghost_rects(hierarchy, level, disjoint=True)
        allc = [r for rl in dcr.values() for r in rl]
        geom = (self.st, self.cst, hierarchy) if self.cst is not None else None
        self.coarse_all = device.RectTable(allc, geom if allc else None)
        # coarse (disjoint from the copies) + copies: one launch when times are synchronised
        self.combined = device.RectTable(allc + list(copies), geom if allc else None)
        shape = hierarchy.level_shape(level)
        ring, phys = _ring_and_physical_all(patches, shape)
        self.full = bool(np.all(covered + phys >= ring))
        self.restrict_to = None      # (coarse store, RectTable) for restriction into level-1
        self._gather = {}            # (boundary, normals, level shape) -> device.GhostPlan

    def job_fill(self, gp):
        """The planned fill regrouped per warp job (built once per plan), or None."""
        jf = self.__dict__.setdefault("_job_fill", {})
        hit = jf.get(id(gp))
        if hit is None or hit[0] is not gp:
            hit = (gp, device.JobFill(self.st, gp) if device.JobFill.usable(self.st) else None)
            jf[id(gp)] = hit
        return hit[1]

    def gather(self, hierarchy, level, ctx):
        """The level's whole fill as one planned gather (built once, on first use)."""
        if not USE_GHOST_PLAN:
            return None
        eq, bd = ctx.equation, ctx.boundary
        key = (device._bc_codes(bd), eq.normal_component(0), eq.normal_component(1) if hierarchy.ndim == 2 else -1,
               tuple(hierarchy.level_shape(level)))
        gp = self._gather.get(key)
        if gp is None:
            if not device.GhostPlan.usable(self.st, self.cst):
                return None
            rects = self.combined if self.coarse_all.n else self.copies
            gp = device.GhostPlan(self.st, rects, self.cst if self.coarse_all.n else None, bd, eq,
                                  hierarchy.level_shape(level))
            self._gather[key] = gp
        return gp

    def valid(self, hierarchy, level) -> bool:
        ps = hierarchy.levels[level - 1] if level - 1 < len(hierarchy.levels) else None
        if ps is not self.plist or len(ps) != self.n or not ps or (ps[0], ps[-1]) != self.ends:
            return False
        if ps[0]._store is not self.st:
            return False
        if level >= 2:
            cl = hierarchy.levels[level - 2]
            if cl is not self.clist or (cl and cl[0]._store is not self.cst):
                return False
        return True


def _plan(hierarchy: PatchHierarchy, level: int) -> LevelPlan:
    plans = hierarchy.__dict__.setdefault("_plans", {})
    pl = plans.get(level)
    if pl is None or not pl.valid(hierarchy, level):
        pl = LevelPlan(hierarchy, level)
        plans[level] = pl
    return pl


def _snap(ctx) -> bool:
    return ctx.variant == _lib.VARIANT_FAST


def _store_time_mode(cst, t, snap: bool = False):
    """(mode, w) shared by every coarse patch, or None when they differ."""
    if cst.time_synced:
        has_old = cst.old is not None and bool(np.all(cst.old_valid))
        probe = cst.patches[0]
        mode = _coarse_time_mode(probe, t, snap) if has_old or probe._host_old is None else None
        return mode
    return None


def fill_level_ghosts(hierarchy: PatchHierarchy, level: int, t: float, ctx: AmrContext, defer: bool = False,
                      substep: int = 0):
    """Coarse interpolation, then same-level copies, then physical boundaries
    (amr.py:479-491), each a batched device launch over the whole level.
    ``defer``: on the fast static-CFL path return the planned fill as step
    arguments instead of launching it (the next launch_step on this level
    runs it; nothing may touch the level in between): ("job", AdjJobFill)
    for a per-warp-job fill, else AdjGhostPlanFillArgs (USE_FUSED_FILL).
    ``substep``: index of this step inside the coarse level's interval."""
    patches = hierarchy.patches(level)
    if not patches:
        return
    pl = _plan(hierarchy, level)
    st = pl.st
    st.sync_in()
    st.prepare_write(full_ghosts=pl.full)
    copies_done = False
    coarse_in = level >= 2 and pl.coarse_all.n
    if coarse_in:
        cst = pl.cst
        cst.sync_in()
        cst.fold_ghosts()
        old_buf = _coarse_old_buffer(cst)
        mw = _store_time_mode(cst, t, _snap(ctx))
    if not coarse_in or mw is not None:
        # level-synchronised times: coarse, copy and physical phases in one gather
        gp = pl.gather(hierarchy, level, ctx)
        if gp is not None:
            if defer and USE_JOB_FILL and gp.n and _static_fast(st, ctx):
                jf = pl.job_fill(gp)
                if jf is not None:
                    st.ghost_src = st.cur
                    if coarse_in and jf.c_base is not None:
                        # coarse values of this interval: computed in its first substep, then cached
                        key = (id(cst), device._ptr(old_buf), device._ptr(cst.buf[cst.cur]), cst.level_time, cst.level_time_old)
                        cmode = 2 if (substep > 0 and jf.cache_key == key) else 1
                        jf.cache_key = key
                        return ("job", jf.args(old_buf, cst.buf[cst.cur], cst, mw[1], mw[0], cmode))
                    return ("job", jf.args())
            if defer and USE_FUSED_FILL and gp.n and _static_fast(st, ctx):
                args = (gp.fill_args(st, old_buf, cst.buf[cst.cur], cst, mw[1], mw[0]) if coarse_in
                        else gp.fill_args(st))
                st.ghost_src = st.cur
                return args
            if coarse_in:
                gp.fill(st, old_buf, cst.buf[cst.cur], cst, mw[1], mw[0])
            else:
                gp.fill(st)
            st.ghost_src = st.cur
            return None
    if coarse_in:
        r = hierarchy.ratio_to_finer(level - 1)
        if mw is not None:
            # disjoint coarse + copy rectangles in one launch
            device.coarse_rects(st, cst, pl.combined, old_buf, cst.buf[cst.cur], hierarchy, r, mw[1], mw[0],
                                copy_src=st.buf[st.cur], copy_patches=st.table)
            copies_done = True
        else:
            groups: dict = {}
            coarse = hierarchy.patches(level - 1)
            for c, rl in pl.crects_by_patch.items():
                groups.setdefault(_coarse_time_mode(coarse[c], t, _snap(ctx)), []).extend(rl)
            for (mode, w), rl in groups.items():
                device.coarse_rects(st, cst, np.array(rl, dtype=_lib.RECT_DTYPE), old_buf, cst.buf[cst.cur],
                                    hierarchy, r, w, mode)
    if pl.copies.n and not copies_done:
        device.copy_rects(st, st, pl.copies, st.buf[st.cur], st.buf[st.cur])
    device.fill_physical(st, ctx.boundary, ctx.equation, hierarchy.level_shape(level))
    st.ghost_src = st.cur


def make_patches(hierarchy: PatchHierarchy, level: int, boxes, ctx: AmrContext, time: float) -> list:
    """make_patch for every (lo, hi) box of a regrid, materials sampled in one batch."""
    from .solver import sample_patches_material
    ps = [Patch(hierarchy.make_spec(level, lo, hi), ctx.equation.m, time=time) for lo, hi in boxes]
    if ps:
        sample_patches_material(ps, ctx.equation, ctx.boundary, hierarchy.level_shape(level))
    return ps


def make_patch(hierarchy: PatchHierarchy, level: int, lo, hi, ctx: AmrContext, time: float) -> Patch:
    spec = hierarchy.make_spec(level, lo, hi)
    p = Patch(spec, ctx.equation.m, time=time)
    sample_patch_material(p, ctx.equation, ctx.boundary, hierarchy.level_shape(level))
    return p


# ---------------------------------------------------------------------------
# restriction (K4)


def _restrict_rects(coarse, fine, r):
    """Overlap of every fine patch's coarsened box with every coarse patch,
    fine patch major then coarse patch ascending (the order of a per-patch
    candidate scan), vectorised over blocks of fine patches."""
    c_lo, c_hi = _boxes(coarse)
    f_lo, f_hi = _boxes(fine)
    nd = c_lo.shape[1]
    out = []
    blk = max(1, (1 << 20) // max(1, len(coarse)))
    for b0 in range(0, len(fine), blk):
        flo, fhi = f_lo[b0:b0 + blk] // r, f_hi[b0:b0 + blk] // r
        lo = np.maximum(flo[:, None, :], c_lo[None])
        hi = np.minimum(fhi[:, None, :], c_hi[None])
        fk, c = np.nonzero(np.all(lo <= hi, axis=2))
        if not len(fk):
            continue
        lo, hi = lo[fk, c], hi[fk, c]
        rc = np.zeros(len(fk), dtype=_lib.RECT_DTYPE)
        rc["dst_patch"], rc["src_patch"] = c, fk + b0
        di, si, ext = lo - c_lo[c], lo * r - f_lo[fk + b0], hi - lo + 1
        rc["di0"], rc["ni"], rc["si0"] = di[:, 0], ext[:, 0], si[:, 0]
        if nd == 2:
            rc["dj0"], rc["nj"], rc["sj0"] = di[:, 1], ext[:, 1], si[:, 1]
        else:
            rc["nj"] = 1
        out.append(rc)
    return np.concatenate(out) if out else np.zeros(0, dtype=_lib.RECT_DTYPE)


def restrict_fine_to_coarse(hierarchy: PatchHierarchy, level: int):
    """Coarse cells covered by level+1 <- mean of their fine children (amr.py:399-450)."""
    fine = hierarchy.patches(level + 1)
    coarse = hierarchy.patches(level)
    if not fine or not coarse:
        return
    r = hierarchy.ratio_to_finer(level)
    fpl = _plan(hierarchy, level + 1)
    cst, fst = fpl.cst, fpl.st
    cst.sync_in()
    fst.sync_in()
    if fpl.restrict_to is None or fpl.restrict_to[0] is not cst:
        rects = _restrict_rects(coarse, fine, r)
        if USE_RESTRICT_PLAN and device.RestrictPlan.usable(cst, fst):
            tab = device.RestrictPlan(cst, fst, rects, r)
        else:
            tab = device.RectTable(rects)
        fpl.restrict_to = (cst, tab)
    cst._unalias()
    device.restrict_rects(cst, fst, fpl.restrict_to[1], r, cst.swe)


# ---------------------------------------------------------------------------
# regrid (flags on device, clustering on host, data movement on device)


def _flag_level(parents, ctx: AmrContext):
    from .adjoint import AdjointFlagging
    if isinstance(ctx.strategy, AdjointFlagging):
        flags, counts = ctx.strategy.evaluate_level(parents)
    else:
        flags = [np.array(ctx.strategy.evaluate(p), dtype=bool) for p in parents]
        counts = None
    out = []
    for p, f in zip(parents, flags):
        f = _apply_regions(np.array(f, dtype=bool), p.spec, p.time, ctx.regions)
        out.append(FlagField(flags=f, lo=p.spec.lo, level=p.spec.level, strategy_name=ctx.strategy.name,
                             time=p.time))
    return out


# adjoint flags post-processed on the device (K5); False: host buffer / mask / clip
USE_DEVICE_FLAG_MASK = True


def _device_level_mask(hierarchy, parent, parents, t, ctx):
    """K3 -> K5 on the device: (clipped, allowed, raw count), or None when the
    strategy is not adjoint flagging or the level store does not match."""
    from .adjoint import AdjointFlagging
    if not USE_DEVICE_FLAG_MASK or not isinstance(ctx.strategy, AdjointFlagging):
        return None
    if len(ctx.regions) > 8:
        return None
    bits, st = ctx.strategy.evaluate_level_bits(parents)
    if len(st.patches) != len(parents) or any(p._store is not st for p in parents):
        return None
    return device.flag_level_mask(st, bits, hierarchy.level_shape(parent), ctx.buffer_cells, ctx.regions, t)


def regrid(hierarchy: PatchHierarchy, level: int, ctx: AmrContext, deepest: int | None = None):
    """Rebuild levels level..deepest from parent flags (amr.py:554-599)."""
    if level < 2:
        raise ValueError("cannot regrid the base level")
    deepest = deepest if deepest is not None else hierarchy.max_levels
    for lev in range(level, deepest + 1):
        parent = lev - 1
        parents = hierarchy.patches(parent)
        while len(hierarchy.levels) < lev:
            hierarchy.levels.append([])
        if not parents:
            hierarchy.levels[lev - 1] = []
            continue
        t = parents[0].time
        fill_level_ghosts(hierarchy, parent, t, ctx)
        dev = _device_level_mask(hierarchy, parent, parents, t, ctx)
        if dev is not None:
            clipped, allowed, raw = dev
        else:
            mask = np.zeros(hierarchy.level_shape(parent), dtype=bool)
            raw = 0
            for ff in _flag_level(parents, ctx):
                raw += int(ff.flags.sum())
                bf = buffer_flags(ff, ctx.buffer_cells)
                sl = _box_slice(ff.lo, tuple(l + n - 1 for l, n in zip(ff.lo, bf.flags.shape)))
                mask[sl] |= bf.flags
            allowed = allowed_region_mask(hierarchy, parent)
            clipped = mask & allowed
        ctx.flagged_per_regrid.append(raw)
        ratio = hierarchy.ratio_to_finer(parent)
        boxes = cluster(clipped, ctx.efficiency, max_edge=max(1, ctx.max_patch_edge // ratio))
        rects = [rb for b in boxes for rb in _allowed_rectangles(b, allowed, clipped)]
        old = hierarchy.patches(lev)
        new = make_patches(hierarchy, lev, [(tuple(l * ratio for l in rb.lo), tuple((h + 1) * ratio - 1 for h in rb.hi))
                                            for rb in rects], ctx, t)
        if new:
            _fill_new_level(hierarchy, lev, new, old, parents, t)
        hierarchy.levels[lev - 1] = new


def _fill_new_level(hierarchy, lev, new, old, parents, t):
    """New interiors: space(-time) interpolation from the parents, then the
    old patches' overlapping interiors (amr.py:504-551), on the device."""
    st = device.LevelStore(new)
    st.set_all_device()            # contents are produced here, nothing to upload
    st.set_level_times(t, None)
    cst = level_store(parents)
    cst.sync_in()
    cst.fold_ghosts()
    r = hierarchy.ratio_to_finer(lev - 1)
    g = new[0].spec.ghost_width
    groups: dict = {}
    crects = _box_overlaps(_lib.RECT_COARSE, new, parents, g, parents[0].spec.ghost_width, r)
    mw = _store_time_mode(cst, t)
    if mw is not None:              # level-synchronised parents: one time mode
        if len(crects):
            groups[mw] = crects
    else:
        for row in crects.tolist():
            groups.setdefault(_coarse_time_mode(parents[row[2]], t), []).append(row)
    old_buf = _coarse_old_buffer(cst)
    for (mode, w), rl in groups.items():
        device.coarse_rects(st, cst, device.RectTable(rl, (st, cst, hierarchy)), old_buf, cst.buf[cst.cur],
                            hierarchy, r, w, mode)
    if old:
        ost = level_store(old)
        ost.sync_in()
        copies = _box_overlaps(_lib.RECT_COPY, new, old, g, old[0].spec.ghost_width, 1)
        if len(copies):
            device.copy_rects(st, ost, copies, ost.buf[ost.cur], st.buf[st.cur])


def _box_overlaps(kind, dst, src, gdst, gsrc, ratio):
    """Rects of every dst box's overlap with the (ratio-refined) src boxes
    (native adj_box_overlaps; same rects, same order as the per-patch scan
    of amr.py:504-551)."""
    import ctypes as C
    nd = dst[0].spec.ndim
    dlo, dhi = (np.ascontiguousarray(a, dtype=np.int32) for a in _boxes(dst))
    slo, shi = (np.ascontiguousarray(a, dtype=np.int32) for a in _boxes(src))
    lib = _lib.load_library()
    cap = max(64, 4 * len(dst) + 4 * len(src))
    while True:
        rects = np.zeros(cap, dtype=_lib.RECT_DTYPE)
        n = _lib.I32()
        rc = lib.adj_box_overlaps(nd, kind, len(dst), dlo.ctypes.data, dhi.ctypes.data, gdst, len(src),
                                  slo.ctypes.data, shi.ctypes.data, gsrc, ratio, rects.ctypes.data, cap, C.byref(n))
        if rc == 0:
            return rects[: n.value]
        if n.value <= cap:
            raise ValueError("adj_box_overlaps: bad arguments")
        cap = n.value


# ---------------------------------------------------------------------------
# the subcycled advance (amr.py:602-644)


def _retry_half_steps(st, slot, patch, dt, ctx):
    """Reference CFL retry: two dt/2 steps from the saved state with the
    ghosts filled at t, no refill in between (amr.py:627-631)."""
    import torch
    from . import solver
    tmp = Patch(patch.spec, patch.num_components, time=patch.time_old)
    tmp.aux = patch.aux
    tmp.state = st.view(slot, "old").cpu().numpy()
    solver.step_patch(tmp, dt / 2.0, ctx.equation, ctx.limiter, variant=ctx.variant)
    solver.step_patch(tmp, dt / 2.0, ctx.equation, ctx.limiter, variant=ctx.variant)
    ts = tmp._store
    g = st.g
    inner = (slice(None),) + (slice(g, -g),) * st.ndim
    st.view(slot)[inner].copy_(ts.view(tmp._slot)[inner])
    del torch


def _fused_restrict(hierarchy, level, pl, ctx, cfl_static):
    """(FusedRestrict, coarse store) when this step may also restrict the
    level into level-1: the finest level's last substep of the interval
    (the caller asks), fast static path, no CFL retry, aligned tiles."""
    if not USE_FUSED_RESTRICT or level < 2 or pl.cst is None or hierarchy.patches(level + 1):
        return None
    _, form, rev = ctx.equation.kernel_spec()
    if cfl_static is None or np.any(cfl_static > 1.0 + 1e-12) or form != _lib.FORM_WAVE or rev:
        return None
    r = hierarchy.ratio_to_finer(level - 1)
    cst, st = pl.cst, pl.st
    if not device.FusedRestrict.usable(cst, st, r):
        return None
    fr = getattr(pl, "fused_restrict", None)
    if fr is None or fr[0] is not cst:
        fr = (cst, device.FusedRestrict(cst, st, _restrict_rects(hierarchy.patches(level - 1),
                                                                 hierarchy.patches(level), r), r))
        pl.fused_restrict = fr
    cst.sync_in()
    cst._unalias()
    return fr[1], cst


def step_level(hierarchy: PatchHierarchy, level: int, dt: float, ctx: AmrContext, prefill=None,
               restrict_into: bool = False) -> bool:
    """save_old + step of every patch of the level in one K1 launch, with the
    reference's per-patch CFL retry and cell-step accounting (amr.py:620-631).

    On the fast path (no dry cells) the CFL bound is the static per-patch
    material speed, so no device->host sync is needed; non-finite results are
    accumulated on the device and raised at the end of the top-level advance.
    ``restrict_into``: this is the last substep of the interval, so the
    restriction into level-1 may run inside the launch; returns whether it did."""
    patches = hierarchy.patches(level)
    pl = _plan(hierarchy, level)
    st = pl.st
    t = patches[0].time
    st.save_old_all()
    st.set_level_times(t, t)
    out = st._free(st.cur)
    static = device.fast_static(st, ctx.equation, ctx.variant)
    if prefill is not None and not static:
        raise RuntimeError("a deferred ghost fill needs the fast static-CFL step")
    job_fill = None
    if isinstance(prefill, tuple):              # ("job", AdjJobFill)
        job_fill, prefill = prefill[1], None
    spec = patches[0].spec
    dtdx = dt / spec.dx
    dtdy = dt / spec.dy if spec.ndim == 2 else 0.0
    cfl_static = None
    if static:
        sm0 = st.static_speed_np()
        cfl_static = np.maximum(sm0[:, 0] * dtdx, sm0[:, 1] * dtdy)
    # the fused restriction rewrites coarse interior cells: only with a fill that does not read the
    # coarse level in this launch (cached coarse values, or no coarse entries)
    may_fuse = prefill is None and (job_fill is None or job_fill.cache_mode == 2 or not job_fill.c_base)
    fused = _fused_restrict(hierarchy, level, pl, ctx, cfl_static) if restrict_into and may_fuse else None
    if fused is not None:
        ctx.__dict__["fused_restrictions"] = ctx.__dict__.get("fused_restrictions", 0) + 1
    smax, bad = device.launch_step(st, dt, ctx.equation, ctx.limiter, ctx.variant, out, accumulate=static,
                                   prefill=prefill, fine_restrict=fused, job_fill=job_fill)
    sm = st.static_speed_np() if static else smax.cpu().numpy()
    cfl = sm[:, 0] * dtdx if spec.ndim == 1 else np.maximum(sm[:, 0] * dtdx, sm[:, 1] * dtdy)
    st.ghost_src = st.cur
    st.cur = out
    st.set_all_device()
    retry = np.flatnonzero(cfl > 1.0 + 1e-12)
    extra = int(sum(int(np.prod(patches[k].spec.shape)) for k in retry))
    ctx.count_step(level, st.total_cells + extra)
    for k in retry:
        _retry_half_steps(st, int(k), patches[int(k)], dt, ctx)
    if static:
        # non-finite flags accumulate in the store (no per-step reduction)
        ctx.__dict__.setdefault("_bad_stores", {})[id(st)] = st
        ctx._bad_pending = True
    else:
        nf = bad.cpu().numpy()
        if np.any(nf):
            raise NumericalBlowupError(f"non-finite state at t={t + dt}")
    return fused is not None


def _raise_pending(ctx):
    """Device-accumulated non-finite flag of the fast path (one sync per
    top-level advance; skipped while a sweep is being captured or shadowed)."""
    if not ctx.__dict__.get("_bad_pending") or ctx.__dict__.get("_defer_checks"):
        return
    ctx._bad_pending = False
    stores = list(ctx.__dict__.get("_bad_stores", {}).values())
    ctx._bad_stores = {}
    hit = False
    for st in stores:
        if st.nonfinite_acc is not None and bool(st.nonfinite_acc.any().item()):
            st.nonfinite_acc.zero_()
            hit = True
    if hit:
        raise NumericalBlowupError("non-finite state during the advance")


def advance_hierarchy(hierarchy: PatchHierarchy, level: int, dt: float, ctx: AmrContext):
    """Advance one level by dt, recursively subcycling finer levels (amr.py:602-644)."""
    depth = ctx.__dict__.get("_depth", 0)
    ctx._depth = depth + 1
    if depth == 0 and _overlap_on(ctx):
        ctx._level_events = {}
        ctx.__dict__.setdefault("_level_streams", {})
    try:
        _advance(hierarchy, level, dt, ctx)
    finally:
        ctx._depth = depth
        if depth == 0 and ctx.__dict__.get("_level_events"):
            for lev in list(ctx._level_events):    # join every side stream into the caller's
                _wait_level(ctx, lev)
            ctx._level_events = {}
    if depth == 0:
        _raise_pending(ctx)


# captured level sweeps (SweepGraph): a parent level's step and its post-step fill run on a side
# stream, concurrently with the first substep of its finer level, which reads only the parent's
# saved pre-step state (coarse time weight 0, amr.py:620-642); every later reader of the parent's
# new state waits for it.  Same launches, same inputs: bitwise equal to the sequential sweep
USE_LEVEL_OVERLAP = os.environ.get("ADJAMR_LEVEL_OVERLAP", "1") == "1"
_OVERLAP_MAX_LEVEL = int(os.environ.get("ADJAMR_OVERLAP_MAX_LEVEL", "99"))   # experiments


def _overlap_on(ctx) -> bool:
    # the in-launch fills (opt-in) read the coarse level's new state from the fine level's step
    # launch, cached interval values included: they keep the sequential capture
    return (bool(ctx.__dict__.get("_overlap")) and not device.SHADOW and ctx.on_level_advanced is None
            and not USE_JOB_FILL and not USE_FUSED_FILL)


def _wait_level(ctx, level):
    """Order the current stream after the in-flight side-stream work of ``level``."""
    ev = ctx.__dict__.get("_level_events", {}).get(level)
    if ev is not None:
        import torch
        torch.cuda.current_stream().wait_event(ev)


def _prefill_needs_coarse_new(hierarchy, level, t, substep, snap) -> bool:
    """Whether the pre-step fill of ``level`` at t may read the coarse level's
    new state (or launch on the coarse store): anything but the first substep
    of an interval with time weight 0 and folded coarse ghosts."""
    if level < 2 or substep > 0:
        return True
    pl = _plan(hierarchy, level)
    cst = pl.cst
    if cst is None or not pl.coarse_all.n:
        return False
    if cst.ghost_src != cst.cur or cst.old is None or not bool(np.all(cst.old_valid)):
        return True
    mw = _store_time_mode(cst, t, snap)
    return mw is None or mw[0] != 0


def _advance(hierarchy, level, dt, ctx, restrict_into: bool = False, substep: int = 0) -> bool:
    """One step of ``level`` and its subcycled finer levels; returns whether
    the restriction of ``level`` into level-1 already ran (fused into the
    step of the interval's last substep of the finest level)."""
    count = ctx.step_counts.get(level, 0)
    if level < hierarchy.max_levels and count > 0 and count % ctx.regrid_interval == 0:
        regrid(hierarchy, level + 1, ctx)
    patches = hierarchy.patches(level)
    if not patches:
        return False
    t = patches[0].time
    ov = _overlap_on(ctx)
    if ov:
        if _prefill_needs_coarse_new(hierarchy, level, t, substep, _snap(ctx)):
            _wait_level(ctx, level - 1)
        elif device.PARAMS is not None and level >= 2 and _plan(hierarchy, level).coarse_all.n:
            # the replayed weight of this fill must stay 0 (SweepGraph checks it per pair)
            ctx._skip_slots.append(len(device.PARAMS.vals))
    pre = fill_level_ghosts(hierarchy, level, t, ctx, defer=True, substep=substep)
    children = level < hierarchy.max_levels and bool(hierarchy.patches(level + 1))
    side = None
    if ov and children and level <= _OVERLAP_MAX_LEVEL:
        import torch
        side = ctx._level_streams.get(level)
        if side is None:
            side = ctx._level_streams[level] = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        side_ctx = torch.cuda.stream(side)
        side_ctx.__enter__()
    elif ov and restrict_into:
        _wait_level(ctx, level - 1)            # a fused restriction writes the coarse new state
    try:
        fused = step_level(hierarchy, level, dt, ctx, prefill=pre, restrict_into=restrict_into)
        t_new = t + dt
        st = patches[0]._store
        st.set_level_times(t_new, t)
        if ctx.on_level_advanced is not None:
            ctx.on_level_advanced(hierarchy, level, t_new)
        ctx.step_counts[level] = count + 1
        if children:
            if side is not None:
                _wait_level(ctx, level - 1)    # the post-step fill reads the coarse new state
            fill_level_ghosts(hierarchy, level, t_new, ctx)
            if side is not None:
                import torch
                ev = torch.cuda.Event()
                ev.record(side)
                ctx._level_events[level] = ev
    finally:
        if side is not None:
            side_ctx.__exit__(None, None, None)
    if children:
        ratio = hierarchy.ratio_to_finer(level)
        done = False
        for k in range(ratio):
            done = _advance(hierarchy, level + 1, dt / ratio, ctx, restrict_into=k == ratio - 1, substep=k)
        if ov:
            _wait_level(ctx, level)
            _wait_level(ctx, level + 1)        # the restriction reads the finer level's last step
        if not done:
            restrict_fine_to_coarse(hierarchy, level)
    return fused


class SweepGraph:
    """CUDA-graph replay of the level sweep (advance_hierarchy without regrid).

    The launch sequence of two coarse steps is fixed once plans exist, and the
    buffer rotation of every level store has period two, so two coarse steps
    are captured once and replayed.  The host bookkeeping (times, step and
    cell counters, buffer roles) is kept exact by re-running the orchestration
    in shadow mode (device.SHADOW: nothing is launched) before every replay.
    Only valid on the static-CFL fast path (fast variant, 2D, no dry cells)
    and while no regrid is due; ``advance`` checks both.

    With USE_LEVEL_OVERLAP the capture puts each parent level's step and
    post-step fill on a side stream: they run concurrently with the first
    substep of the finer level (which reads the parent's saved state only),
    and the graph's edges are exactly the sweep's data dependencies."""

    def __init__(self, hierarchy: PatchHierarchy, dt: float, ctx: AmrContext):
        import torch
        self.h, self.dt, self.ctx = hierarchy, dt, ctx
        if ctx.variant != _lib.VARIANT_FAST or hierarchy.ndim != 2:
            raise ValueError("SweepGraph needs the fast 2D path")
        for _ in range(2):                      # warm-up: plans, stores, buffers, caches
            advance_hierarchy(hierarchy, 1, dt, ctx)
        for lev in range(1, hierarchy.num_levels() + 1):
            st = _plan(hierarchy, lev).st
            if not device.fast_static(st, ctx.equation, ctx.variant):
                raise ValueError("SweepGraph needs the static-CFL fast path on every level")
            for i in range(st.NBUF):
                st._ensure_buf(i)
        torch.cuda.synchronize()
        self._levels = [lev for lev in range(1, hierarchy.num_levels() + 1) if hierarchy.patches(lev)]
        self._stores = {lev: _plan(hierarchy, lev).st for lev in self._levels}
        self.params = device.ParamSlots()
        # the overlapped capture (parent steps on side streams); when some first-substep fill of
        # it skipped the wait for its coarse level, also a sequential one, replayed for a pair
        # whose weight at such a fill is not 0
        self.graph, self.skip_slots = self._capture(USE_LEVEL_OVERLAP)
        self.graph_seq = None
        if self.skip_slots:                     # captured, not run: the bookkeeping is restored
            book = self._book()
            self.graph_seq = self._capture(False, replay=False)[0]
            self._restore(book)
        self.seq_replays = 0
        # lite shadow: the host bookkeeping of a pair (level times, counters,
        # time-weight slots) without the orchestration; trusted only after it
        # reproduced a full shadow pair exactly (_shadow_pair)
        self.lite_ok = None
        self._coarse_in = {lev: lev >= 2 and bool(_plan(hierarchy, lev).coarse_all.n) for lev in self._levels}
        self._fused_per_pair = None

    def _capture(self, overlap, replay=True):
        """Capture two coarse steps, then replay them once (the device catches
        up with the captured steps' bookkeeping); returns (graph, slots whose
        weight must be -1 for a replay)."""
        import torch
        h, ctx = self.h, self.ctx
        before = self._roles()
        graph = torch.cuda.CUDAGraph()
        self.params.rewind()
        ctx._defer_checks = True
        ctx._overlap = overlap
        ctx._skip_slots = []
        ctx.__dict__.setdefault("_level_streams", {})
        for lev in range(1, h.num_levels() + 1):   # side streams exist before the capture
            ctx._level_streams.setdefault(lev, torch.cuda.Stream())
        device.PARAMS = self.params
        try:
            with torch.cuda.graph(graph):
                for _ in range(2):
                    advance_hierarchy(h, 1, self.dt, ctx)
        finally:
            ctx._defer_checks = False
            ctx._overlap = False
            device.PARAMS = None
        skip = list(ctx._skip_slots)
        ctx._skip_slots = []
        self.params.upload()
        if self._roles() != before:
            raise RuntimeError("level sweep is not 2-periodic; cannot replay")
        if replay:
            graph.replay()
        return graph, skip

    def _book(self):
        ctx = self.ctx
        return ({lev: (st.time_synced, st.level_time, st.level_time_old) for lev, st in self._stores.items()},
                dict(ctx.step_counts), dict(ctx.cell_steps), ctx.__dict__.get("fused_restrictions", 0))

    def _restore(self, book):
        times, counts, cells, fused = book
        for lev, (synced, t, t_old) in times.items():
            self._stores[lev].set_level_times(t, t_old)
        self.ctx.step_counts.clear(); self.ctx.step_counts.update(counts)
        self.ctx.cell_steps.clear(); self.ctx.cell_steps.update(cells)
        self.ctx.__dict__["fused_restrictions"] = fused

    def _lite_pair(self) -> list:
        """Two coarse steps of the _advance recursion on the host bookkeeping
        only: the same float operations on the level times (t + dt, dt / r,
        _store_time_mode), the same counter updates; returns the slot values
        in take() order."""
        h, ctx, st_of = self.h, self.ctx, self._stores
        vals = []

        def fill(lev, t):
            if self._coarse_in.get(lev):
                mode, w = _store_time_mode(st_of[lev - 1], t, _snap(ctx))
                vals.append(w if mode == 1 else -1.0)

        def adv(lev, dt):
            count = ctx.step_counts.get(lev, 0)
            st = st_of[lev]
            t = st.level_time
            fill(lev, t)
            st.set_level_times(t, t)
            ctx.count_step(lev, st.total_cells)
            t_new = t + dt
            st.set_level_times(t_new, t)
            ctx.step_counts[lev] = count + 1
            if lev < h.max_levels and (lev + 1) in st_of:
                fill(lev, t_new)
                ratio = h.ratio_to_finer(lev)
                for _ in range(ratio):
                    adv(lev + 1, dt / ratio)

        for _ in range(2):
            adv(1, self.dt)
        ctx.__dict__["fused_restrictions"] = ctx.__dict__.get("fused_restrictions", 0) + self._fused_per_pair
        for st in st_of.values():
            ctx.__dict__.setdefault("_bad_stores", {})[id(st)] = st
        return vals

    def _full_shadow(self):
        device.SHADOW = True
        device.PARAMS = self.params
        self.params.rewind()
        self.ctx._defer_checks = True
        try:
            for _ in range(2):
                advance_hierarchy(self.h, 1, self.dt, self.ctx)
        finally:
            device.SHADOW = False
            device.PARAMS = None
            self.ctx._defer_checks = False

    def _shadow_pair(self):
        """Host bookkeeping of the next replayed pair.  The first pair runs
        both the lite shadow and the full one (from the same bookkeeping) and
        keeps the lite one only if times, counters and slot values agree
        exactly; otherwise every pair runs the full shadow."""
        if self.lite_ok:
            self.params.vals = self._lite_pair()
            return
        if (self.lite_ok is None and self.ctx.on_level_advanced is None and not USE_JOB_FILL and
                all(st.time_synced for st in self._stores.values())):
            before = self._book()
            f0 = before[3]
            self._fused_per_pair = 0
            try:
                lite_vals = self._lite_pair()
                lite_book = self._book()
            except Exception:       # noqa: BLE001 -- any mismatch disables the lite path
                lite_vals, lite_book = None, None
            self._restore(before)
            self._full_shadow()
            full_book = self._book()
            self._fused_per_pair = full_book[3] - f0
            if lite_book is not None:
                lite_book = lite_book[:3] + (lite_book[3] + self._fused_per_pair,)
            self.lite_ok = lite_vals is not None and lite_vals == self.params.vals and lite_book == full_book
            return
        self.lite_ok = False
        self._full_shadow()

    def _roles(self):
        out = []
        for lev in range(1, self.h.num_levels() + 1):
            st = _plan(self.h, lev).st
            out.append((id(st), st.cur, st.old, st.ghost_src))
        return out

    def _regrid_due(self, steps: int) -> bool:
        c = self.ctx.step_counts
        for lev in range(1, self.h.max_levels):
            n = c.get(lev, 0)
            per = 1
            for l2 in range(1, lev):
                per *= self.h.ratio_to_finer(l2)
            if any((n + k) > 0 and (n + k) % self.ctx.regrid_interval == 0 for k in range(steps * per)):
                return True
        return False

    def advance(self, coarse_steps: int):
        """Advance by an even number of coarse steps (graph replays)."""
        if coarse_steps % 2:
            raise ValueError("SweepGraph advances in pairs of coarse steps")
        if self._regrid_due(coarse_steps):
            raise ValueError("a regrid falls inside the replayed steps")
        for _ in range(coarse_steps // 2):
            self._shadow_pair()
            self.params.upload()
            g = self.graph
            if self.graph_seq is not None and any(self.params.vals[i] != -1.0 for i in self.skip_slots):
                g = self.graph_seq
                self.seq_replays += 1
            g.replay()
        self.ctx._bad_pending = True
        _raise_pending(self.ctx)
