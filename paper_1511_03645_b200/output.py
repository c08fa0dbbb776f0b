"""Output path on the device: only scalars and gauge values
cross to the host at output times; snapshots download each level once.

  evaluate_J            adjoint.py:299-336 (+ _uncovered_mask 280-296)
  GaugeSeries,
  record_gauge(s),
  write_gauge           runio.py:205-233
  write_snapshot        runio.py:43-77 (text format, 17 significant digits)

evaluate_J computes every cell's inner product with the reference's
arithmetic (K3's interpolation, -fmad=false) and sums per CUDA block in a
fixed order; the per-patch sums are combined on the host in patch order and
scaled by the cell area as the reference does, so the result agrees with the
reference to a few ulps of sum |terms| (not bitwise: numpy sums pairwise).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib, device
from .adjoint import AdjointSnapshotStore, _adjoint_geometry
from .geometry import OutOfRangeError, PatchHierarchy, UniformField

_THREADS = 256
_CELLS_PER_THREAD = 4


def _qhat_source(store_or_phi, t):
    """(ring, snap code, w, origin, dx, dy, shape) of the adjoint field at t:
    interpolate_time (adjoint.py:98-110) encoded for the kernel, or a fixed
    UniformField (e.g. the functional weight) as a one-snapshot ring."""
    import torch
    if isinstance(store_or_phi, AdjointSnapshotStore):
        st = store_or_phi
        ring = st.ring()
        origin, adx, ady, shape = _adjoint_geometry(st)
        times = np.asarray(st.times, dtype=float)
        eps = 1e-9 * max(abs(times[-1]), 1.0)
        if t <= times[0] + eps:
            k, w = -1, 0.0
        elif t >= times[-1] - eps:
            k, w = -len(times), 0.0
        else:
            n = int(np.searchsorted(times, t) - 1)
            k, w = n, float((t - times[n]) / (times[n + 1] - times[n]))
        return ring, k, w, tuple(origin), adx, ady, tuple(shape)
    if isinstance(store_or_phi, UniformField):
        f = store_or_phi
        ring = torch.from_numpy(np.ascontiguousarray(f.values, dtype=float)[None]).to("cuda")
        return ring, -1, 0.0, tuple(f.origin), f.dx, f.dy, tuple(f.values.shape[1:])
    raise TypeError(f"cannot evaluate J against a {type(store_or_phi).__name__}")


def _uniform_as_store(field_: UniformField):
    """A one-patch device view of a UniformField (no ghosts) for the kernel."""
    import torch
    vals = np.ascontiguousarray(field_.values, dtype=float)
    m = vals.shape[0]
    shape = vals.shape[1:]
    nx = shape[0]
    ny = shape[1] if len(shape) == 2 else 1
    tab = np.zeros(1, dtype=_lib.PATCH_DTYPE)
    tab[0] = (0, 0, nx, ny, ny if len(shape) == 2 else 1, 0, 0, 0, 0, 0)
    q = torch.from_numpy(vals.reshape(m, -1).copy()).to("cuda")
    return q, device._dev_table(tab), nx * ny, m


def _launch_functional(q, table, npatch, comp_stride, ghost, ndim, m, max_cells, geom, src, finer=None,
                       level_shape=(1, 1), ratio=1):
    import torch
    ring, k, w, a_origin, adx, ady, ashape = src
    bx = max(1, -(-max_cells // (_THREADS * _CELLS_PER_THREAD)))
    partial = torch.empty(npatch * bx, dtype=torch.float64, device="cuda")
    status = torch.empty(1, dtype=torch.int32, device="cuda")
    covered = None
    a = _lib.AdjFunctionalArgs()
    a.q = device._ptr(q)
    a.patches = device._ptr(table)
    a.ring = device._ptr(ring)
    if finer is not None:
        ftab, nfiner = finer
        covered = torch.empty(int(level_shape[0]) * int(level_shape[1]), dtype=torch.uint8, device="cuda")
        a.finer, a.nfiner, a.covered, a.ratio = device._ptr(ftab), nfiner, device._ptr(covered), ratio
    a.partial = device._ptr(partial)
    a.status = device._ptr(status)
    a.comp_stride = comp_stride
    a.npatch, a.ndim, a.m, a.ghost = npatch, ndim, m, ghost
    a.nxa = ashape[0]
    a.nya = ashape[1] if ndim == 2 else 1
    a.level_nx, a.level_ny = int(level_shape[0]), int(level_shape[1])
    a.blocks_x = bx
    a.snap, a.w = k, w
    a.origin_x, a.origin_y, a.dx, a.dy = geom
    a.a_origin_x = a_origin[0]
    a.a_origin_y = a_origin[1] if ndim == 2 else 0.0
    a.a_dx, a.a_dy = adx, ady
    _lib.check(_lib.lib().adj_functional(_lib.C.byref(a)), "adj_functional")
    if int(status.item()):
        raise OutOfRangeError("interpolation point outside the adjoint domain")
    return partial.cpu().numpy().reshape(npatch, bx)


def evaluate_J(source, store_or_phi, t: float) -> float:
    """Discrete inner-product integral over the finest available cells
    (adjoint.py:299-336).  ``source``: PatchHierarchy (device level stores)
    or UniformField; ``store_or_phi``: AdjointSnapshotStore (interpolated in
    time to t) or a UniformField such as the functional weight."""
    from .solver import level_store
    src = _qhat_source(store_or_phi, t)
    if isinstance(source, UniformField):
        q, tab, ncell, m = _uniform_as_store(source)
        nd = source.ndim
        geom = (source.origin[0], source.origin[1] if nd == 2 else 0.0, source.dx, source.dy if nd == 2 else 0.0)
        part = _launch_functional(q, tab, 1, ncell, 0, nd, m, ncell, geom, src)
        s = 0.0
        for v in part[0]:
            s = s + float(v)
        return float(s * (source.dx if nd == 1 else source.dx * source.dy))
    if not isinstance(source, PatchHierarchy):
        raise TypeError(f"cannot evaluate J on a {type(source).__name__}")
    nd = source.ndim
    total = 0.0
    for level in range(1, source.num_levels() + 1):
        patches = source.patches(level)
        if not patches:
            continue
        st = level_store(patches)
        st.sync_in()
        wx, wy = source.widths(level)
        area = wx if nd == 1 else wx * wy
        finer = source.patches(level + 1) if level < source.num_levels() else []
        ftab = None
        shape = source.level_shape(level)
        if finer:
            t_np = np.zeros(len(finer), dtype=_lib.PATCH_DTYPE)
            for k, fp in enumerate(finer):
                s = fp.spec
                t_np[k] = (0, 0, s.shape[0], s.shape[1] if nd == 2 else 1, 1, s.lo[0], s.lo[1] if nd == 2 else 0,
                           0, 0, 0)
            ftab = (device._dev_table(t_np), len(finer))
        org = source.origin
        geom = (org[0], org[1] if nd == 2 else 0.0, wx, wy if nd == 2 else 0.0)
        max_cells = max(int(np.prod(p.spec.shape)) for p in patches)
        part = _launch_functional(st.buf[st.cur], st.table, len(st.patches), st.plane, st.g, nd, st.m, max_cells,
                                  geom, src, finer=ftab, level_shape=(shape[0], shape[1] if nd == 2 else 1),
                                  ratio=source.ratio_to_finer(level) if finer else 1)
        for p in patches:
            s = 0.0
            for v in part[p._slot]:
                s = s + float(v)
            total += float(s * area)
    return total


# ---------------------------------------------------------------------------
# gauges

@dataclass
class GaugeSeries:
    gauge_id: int
    location: tuple[float, ...]
    times: list = field(default_factory=list)
    values: list = field(default_factory=list)     # one (m,) vector per time

    def as_arrays(self):
        return np.asarray(self.times), np.asarray(self.values)


def _axis_stencil(x, lo_phys, width, n):
    """_axis_weights (geometry.py:248-260) for one coordinate -> (i0, i1, w)."""
    s = (float(x) - lo_phys) / width - 0.5
    fl = np.floor(s)
    i0 = int(fl)
    w = float(s - fl)
    if i0 < 0:
        w = 0.0
    elif i0 > n - 2:
        w = 1.0
    i0 = min(max(i0, 0), max(n - 2, 0))
    if n == 1:
        w = 0.0
    return i0, min(i0 + 1, n - 1), w


def record_gauges(hierarchy: PatchHierarchy, series_list, t: float):
    """record_gauge for many gauges: one K3-gauge launch per level store,
    one small D2H (runio.py:217-226: finest patch, interior-only stencil)."""
    import torch
    from .solver import level_store
    by_store: dict = {}
    for s in series_list:
        p = hierarchy.finest_patch_at(s.location)
        if p is None:
            continue
        st = level_store(hierarchy.patches(p.spec.level))
        by_store.setdefault(id(st), (st, []))[1].append((s, p))
    for st, items in by_store.values():
        st.sync_in()
        nd = st.ndim
        rows = np.zeros(len(items), dtype=_lib.GAUGE_DTYPE)
        for k, (s, p) in enumerate(items):
            spec = p.spec
            off, NX, NY, pitch = st.boxes[p._slot]
            g = st.g
            base = off + g * pitch + (g if nd == 2 else 0)
            i0, i1, wx = _axis_stencil(s.location[0], spec.origin[0] + spec.lo[0] * spec.dx, spec.dx, spec.shape[0])
            j0 = j1 = 0
            wy = 0.0
            if nd == 2:
                j0, j1, wy = _axis_stencil(s.location[1], spec.origin[1] + spec.lo[1] * spec.dy, spec.dy,
                                           spec.shape[1])
            rows[k] = (base, pitch, i0, i1, j0, j1, 0, wx, wy)
        gt = device._dev_table(rows)
        out = torch.empty(len(items) * st.m, dtype=torch.float64, device="cuda")
        a = _lib.AdjGaugeArgs()
        a.q = device._ptr(st.buf[st.cur])
        a.gauges = device._ptr(gt)
        a.out = device._ptr(out)
        a.comp_stride = st.plane
        a.ngauge, a.ndim, a.m = len(items), nd, st.m
        _lib.check(_lib.lib().adj_gauges(_lib.C.byref(a)), "adj_gauges")
        vals = out.cpu().numpy().reshape(len(items), st.m)
        for (s, _), v in zip(items, vals):
            s.times.append(float(t))
            s.values.append(v.copy())


def record_gauge(hierarchy: PatchHierarchy, series: GaugeSeries, t: float):
    """Append the interpolated state at the gauge from the finest cover."""
    record_gauges(hierarchy, [series], t)


def _fmt(x: float) -> str:
    return format(float(x), ".17g")


def write_gauge(series: GaugeSeries, path: str):
    with open(path, "w") as f:
        loc = ",".join(_fmt(v) for v in series.location)
        f.write(f"# gauge {series.gauge_id} at {loc}\n")
        for t, v in zip(series.times, series.values):
            f.write(",".join([_fmt(t)] + [_fmt(x) for x in v]) + "\n")


# ---------------------------------------------------------------------------
# snapshots

@dataclass
class PatchRecord:
    level: int
    lo: tuple[int, ...]
    hi: tuple[int, ...]
    dx: float
    dy: float
    time: float
    values: np.ndarray            # (m, nx[, ny])


def snapshot_records(obj) -> list[PatchRecord]:
    """Patch records ordered by level then corner (runio.py:47-64); each
    level's interiors come from ONE device-to-host copy of its store."""
    from .solver import level_store
    if isinstance(obj, UniformField):
        nd = obj.ndim
        return [PatchRecord(level=1, lo=(0,) * nd, hi=tuple(n - 1 for n in obj.shape), dx=obj.dx, dy=obj.dy,
                            time=obj.time, values=obj.values)]
    if not isinstance(obj, PatchHierarchy):
        raise TypeError(f"cannot snapshot a {type(obj).__name__}")
    recs = []
    for level in range(1, obj.num_levels() + 1):
        patches = obj.patches(level)
        if not patches:
            continue
        wx, wy = obj.widths(level)
        st = level_store(patches)
        st.sync_in()
        host = st.buf[st.cur].cpu().numpy()
        g = st.g
        for p in sorted(patches, key=lambda q: q.spec.lo):
            off, NX, NY, pitch = st.boxes[p._slot]
            blk = np.lib.stride_tricks.as_strided(host[off:], (st.m, NX, NY), (8 * st.plane, 8 * pitch, 8))
            vals = blk[:, g:NX - g, g:NY - g] if st.ndim == 2 else blk[:, g:NX - g, 0]
            recs.append(PatchRecord(level=level, lo=p.spec.lo, hi=p.spec.hi, dx=wx, dy=wy, time=p.time,
                                    values=np.array(vals)))
    return recs


def write_snapshot(obj, path: str):
    """Plain-text snapshot in the reference format (runio.py:66-77)."""
    with open(path, "w") as f:
        for r in snapshot_records(obj):
            lo = ",".join(str(i) for i in r.lo)
            hi = ",".join(str(i) for i in r.hi)
            f.write(f"patch level={r.level} lo={lo} hi={hi} dx={_fmt(r.dx)} "
                    f"dy={_fmt(r.dy)} time={_fmt(r.time)} m={r.values.shape[0]}\n")
            flat = r.values.reshape(r.values.shape[0], -1)
            for col in range(flat.shape[1]):
                f.write(" ".join(_fmt(v) for v in flat[:, col]) + "\n")
