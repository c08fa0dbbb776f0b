"""Adjoint snapshot ring in HBM and inner-product flagging (K3).

Drop-in for the reference's adjoint.py (/root/reference/pkg/src/adjamr/
adjoint.py): the snapshot store keeps its host API (times, fields, window,
wet) and mirrors the fields once into a device ring (N, m, nxa[, nya]) fp64;
``inner_product_field`` / ``inner_product_flags`` / ``AdjointFlagging`` run
the K3 kernel, which emits bit-packed flags plus raw counts.  The window
query and time weights are host arithmetic; ``solve_adjoint`` runs the
reversed f-wave system with the device K1/K2 loop.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib, device
from .geometry import OutOfRangeError, Patch, PatchHierarchy, UniformField


class ConfigurationError(RuntimeError):
    """The adjoint machinery was invoked without a required ingredient (adjoint.py:24)."""


class EmptyFunctionalError(ValueError):
    """The functional's region of interest misses every cell centre (adjoint.py:28)."""


@dataclass(frozen=True)
class FunctionalSpec:
    kind: str
    bounds: tuple[float, ...]
    weights: tuple[float, ...]

    def __post_init__(self):
        if self.kind not in ("box", "disk"):
            raise ValueError(f"unknown functional shape {self.kind!r}")
        if not all(np.isfinite(w) for w in self.weights):
            raise ValueError("functional weights must be finite")

    def indicator(self, x, y=None):
        if self.kind == "box":
            if y is None:
                return (x >= self.bounds[0]) & (x <= self.bounds[1])
            x1, x2, y1, y2 = self.bounds
            return (x >= x1) & (x <= x2) & (y >= y1) & (y <= y2)
        xc, yc, r = self.bounds
        return (x - xc) ** 2 + (y - yc) ** 2 <= r ** 2


@dataclass(frozen=True)
class TimeWindow:
    t_start: float
    t_final: float

    def __post_init__(self):
        if self.t_start > self.t_final:
            raise ValueError("t_start must be <= t_final")

    @property
    def span(self) -> float:
        return self.t_final - self.t_start


@dataclass
class AdjointSnapshotStore:
    """Snapshots labelled by forward time, ascending (adjoint.py:72-110), plus
    their device ring (built lazily, kept while the store is alive)."""

    times: np.ndarray
    fields: list
    window: TimeWindow
    wet: np.ndarray | None = None
    _ring: object = field(default=None, repr=False, compare=False)
    _wet_dev: object = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        self.times = np.asarray(self.times, dtype=float)
        d = np.diff(self.times)
        if len(d) and (np.any(d <= 0) or np.ptp(d) > 1e-9 * max(d[0], 1.0)):
            raise ValueError("snapshot times must be strictly increasing and uniform")

    @property
    def dt_snap(self) -> float:
        return float(self.times[1] - self.times[0]) if len(self.times) > 1 else 0.0

    @property
    def grid(self) -> UniformField:
        return self.fields[0]

    def phi(self) -> UniformField:
        return self.fields[-1]

    def interpolate_time(self, t: float) -> UniformField:
        """Host restatement kept for API parity (adjoint.py:98-110)."""
        eps = 1e-9 * max(abs(self.times[-1]), 1.0)
        if t <= self.times[0] + eps:
            return self.fields[0]
        if t >= self.times[-1] - eps:
            return self.fields[-1]
        n, w = _bracket(self.times, t)
        f = self.fields[n]
        return UniformField(values=(1 - w) * f.values + w * self.fields[n + 1].values,
                            origin=f.origin, dx=f.dx, dy=f.dy, time=t)

    # device mirror -------------------------------------------------------
    def ring(self):
        import torch
        if self._ring is None:
            vals = np.stack([np.asarray(f.values, dtype=float) for f in self.fields])
            self._ring = torch.from_numpy(vals).to("cuda")
            if self.wet is not None:
                self._wet_dev = torch.from_numpy(np.ascontiguousarray(self.wet, dtype=np.uint8)).to("cuda")
        return self._ring

    @classmethod
    def from_device(cls, times, ring, origin, dx, dy, window, wet=None):
        """Store whose snapshots already live in HBM (no host copy until asked)."""
        s = cls.__new__(cls)
        s.times = np.asarray(times, dtype=float)
        s.window = window
        s.wet = wet
        s._ring = ring
        s._wet_dev = None
        if wet is not None:
            import torch
            s._wet_dev = torch.from_numpy(np.ascontiguousarray(wet, dtype=np.uint8)).to("cuda")
        s.fields = _LazyFields(ring, s.times, origin, dx, dy)
        return s


class _LazyFields(list):
    """List-like view of device snapshots, downloaded per access."""

    def __init__(self, ring, times, origin, dx, dy):
        super().__init__()
        self._ring, self._times, self._o, self._dx, self._dy = ring, times, origin, dx, dy

    def __len__(self):
        return int(self._ring.shape[0])

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        if k < 0:
            k += len(self)
        return UniformField(values=self._ring[k].cpu().numpy(), origin=self._o, dx=self._dx, dy=self._dy,
                            time=float(self._times[k]))

    def __iter__(self):
        for k in range(len(self)):
            yield self[k]


def _bracket(times, t):
    n = int(np.searchsorted(times, t) - 1)
    return n, (t - times[n]) / (times[n + 1] - times[n])


def window_indices(t: float, window: TimeWindow, times) -> list[int]:
    """query_window_times on a bare time array (adjoint.py:192-214)."""
    times = np.asarray(times, dtype=float)
    dts = float(times[1] - times[0]) if len(times) > 1 else 0.0
    eps = 1e-9 * max(dts, abs(float(times[-1])), 1.0)
    if t > times[-1] + eps:
        return []
    upper = min(t + window.span, window.t_final)
    sel = np.flatnonzero((times >= t - eps) & (times <= upper + eps))
    out = [int(k) for k in sel]
    if sel.size == 0 or times[sel[0]] > t + eps:
        lower = np.flatnonzero(times < t - eps)
        if lower.size:
            out.insert(0, int(lower[-1]))
    if sel.size == 0 or times[sel[-1]] < upper - eps:
        higher = np.flatnonzero(times > upper + eps)
        if higher.size:
            out.append(int(higher[0]))
    return out


def query_window_times(t: float, window: TimeWindow, store: AdjointSnapshotStore) -> list[int]:
    return window_indices(t, window, store.times)


def interp_window(t: float, window: TimeWindow, times) -> tuple[list[int], list[float]]:
    """Time-interpolated window (north_star; D1): the adjoint interpolated
    linearly in time at t and at min(t+span, t_final), plus every snapshot
    strictly between.  Encoded for K3 mode 1: k >= 0 blends k, k+1 with w;
    k < 0 is snapshot -k-1 unblended."""
    times = np.asarray(times, dtype=float)
    eps = 1e-9 * max(abs(times[-1]), 1.0)
    upper = min(t + window.span, window.t_final)
    ks, ws = [], []

    def point(tt):
        if tt <= times[0] + eps:
            ks.append(-1); ws.append(0.0)
        elif tt >= times[-1] - eps:
            ks.append(-len(times)); ws.append(0.0)
        else:
            n, w = _bracket(times, tt)
            ks.append(n); ws.append(float(w))
    if t > times[-1] + eps:
        return [], []
    point(t)
    for k in np.flatnonzero((times > t + eps) & (times < upper - eps)):
        ks.append(-int(k) - 1); ws.append(0.0)
    if upper > t + eps:
        point(upper)
    return ks, ws


def _adjoint_geometry(store):
    g = store.grid if not isinstance(store.fields, _LazyFields) else None
    if g is not None:
        return g.origin, g.dx, g.dy, g.values.shape[1:]
    f = store.fields
    return f._o, f._dx, f._dy, tuple(store._ring.shape[2:])


def flag_level(patches: list[Patch], t: float, store: AdjointSnapshotStore, window: TimeWindow,
               tolerance: float, want_best: bool = False, time_interp: bool = False, device_bits: bool = False,
               variant: int | None = None):
    """K3 over every patch of a level in one launch.  Returns (flags: list of
    bool arrays, raw counts: list of int, best: list of arrays or None);
    ``device_bits``: (packed flag words on the device, level store) instead.
    ``variant``: VARIANT_EXACT (default; the reference's arithmetic, bitwise)
    or VARIANT_FAST (multi-snapshot windows with FMA interpolation; flags
    identical except for cells within 1e-12 relative of the tolerance)."""
    if store is None:
        raise ConfigurationError("adjoint flagging requires a snapshot store")
    from .solver import level_store
    st = patches[0]._store
    if st is None or any(p._store is not st for p in patches):
        st = level_store(patches)
    st.sync_in()
    slots = [p._slot for p in patches]
    ring = store.ring()
    origin, adx, ady, ashape = _adjoint_geometry(store)
    if time_interp:
        idx, w = interp_window(t, window, store.times)
    else:
        idx, w = query_window_times(t, window, store), None
    spec = patches[0].spec
    bits, counts, best, status = device.launch_flag(
        st, ring, ashape, origin, adx, ady, spec.origin, spec.dx, spec.dy if spec.ndim == 2 else 0.0,
        idx, tolerance, adj_wet=store._wet_dev if spec.ndim == 2 else None, interp_w=w, want_best=want_best,
        variant=variant)
    if int(status[0].item()):
        raise OutOfRangeError("interpolation point outside the adjoint domain")
    if device_bits:
        return bits, st
    words = bits[: max(st.flag_words, 1)].cpu().numpy().view(np.uint32)
    cnt = counts[: len(st.patches)].cpu().numpy()[slots]
    flags = []
    for k, p in zip(slots, patches):
        n = int(np.prod(p.spec.shape))
        fw = int(st.table_np["flag_word"][k])
        wb = words[fw: fw + (n + 31) // 32]
        bitsk = np.unpackbits(wb.view(np.uint8), bitorder="little")[:n].astype(bool)
        flags.append(bitsk.reshape(p.spec.shape))
    bests = None if best is None else [best[k].cpu().numpy().reshape(p.spec.shape) for k, p in zip(slots, patches)]
    return flags, [int(c) for c in cnt], bests


def inner_product_field(patch: Patch, t: float, store: AdjointSnapshotStore, window: TimeWindow):
    """Windowed max of |qhat . q| per interior cell (adjoint.py:227-249), on the device."""
    _, _, best = flag_level([patch], t, store, window, np.inf, want_best=True)
    return best[0]


def inner_product_flags(patch: Patch, t: float, store: AdjointSnapshotStore, window: TimeWindow,
                        tolerance: float):
    """Cells whose windowed inner product exceeds tolerance (adjoint.py:252-257)."""
    from .amr import FlagField
    flags, _, _ = flag_level([patch], t, store, window, tolerance)
    return FlagField(flags=flags[0], lo=patch.spec.lo, level=patch.spec.level, strategy_name="adjoint", time=t)


def build_phi(functional: FunctionalSpec, origin, widths, shape) -> UniformField:
    """Weight field (adjoint.py:113-129): weight x indicator at cell centres."""
    m = len(functional.weights)
    xs = origin[0] + (np.arange(shape[0]) + 0.5) * widths[0]
    if len(shape) == 1:
        ind = functional.indicator(xs)
    else:
        ys = origin[1] + (np.arange(shape[1]) + 0.5) * widths[1]
        ind = functional.indicator(xs[:, None], ys[None, :])
    if not np.any(ind):
        raise EmptyFunctionalError("functional region contains no cell centers")
    vals = np.zeros((m, *shape))
    for k, w in enumerate(functional.weights):
        vals[k] = w * ind
    return UniformField(values=vals, origin=tuple(origin), dx=widths[0], dy=widths[1] if len(shape) == 2 else 0.0)


def solve_adjoint(equation, boundary, functional: FunctionalSpec, window: TimeWindow, domain_xlim, domain_ylim,
                  grid_shape, t0: float = 0.0, dt_snap: float | None = None, *, courant_target: float = 0.9,
                  limiter: str = "MC", log=None, keep_on_device: bool = False) -> AdjointSnapshotStore:
    """Reversed f-wave adjoint solve on a uniform grid (adjoint.py:132-189):
    the device integrate loop writes each snapshot straight into the HBM ring."""
    import torch
    from . import solver
    duration = window.t_final - t0
    if duration <= 0:
        raise ValueError("t_final must exceed t0")
    if dt_snap is None:
        dt_snap = duration / 64.0
    nsnap = max(1, round(duration / dt_snap))
    snap_times = np.linspace(0.0, duration, nsnap + 1)
    nd = 1 if domain_ylim is None else 2
    origin = (domain_xlim[0],) if nd == 1 else (domain_xlim[0], domain_ylim[0])
    wx = (domain_xlim[1] - domain_xlim[0]) / grid_shape[0]
    wy = 0.0 if nd == 1 else (domain_ylim[1] - domain_ylim[0]) / grid_shape[1]
    phi = build_phi(functional, origin, (wx, wy), grid_shape)
    if np.all(phi.values == 0.0) and log is not None:
        log("warning: functional weight field is identically zero")
    rev = equation.adjoint().reversed()
    h = PatchHierarchy(xlim=tuple(domain_xlim), ylim=None if nd == 1 else tuple(domain_ylim),
                       base_shape=tuple(grid_shape), ratios=[])
    spec = h.make_spec(1, (0,) * nd, tuple(n - 1 for n in grid_shape))
    patch = Patch(spec, rev.m, time=0.0)
    solver.sample_patch_material(patch, rev, boundary, tuple(grid_shape))
    patch.interior()[...] = phi.values
    st = solver.store_of(patch)
    ring = torch.zeros((nsnap + 1, rev.m, *grid_shape), dtype=torch.float64, device="cuda")
    labels = []
    g = spec.ghost_width
    inner = (slice(None),) + (slice(g, -g),) * nd

    def on_output(t_rev, p):
        k = len(labels)
        st.sync_in()
        st.fold_ghosts()
        ring[len(ring) - 1 - k].copy_(st.view(p._slot)[inner])
        labels.append(t_rev)

    solver.integrate_patch(patch, rev, boundary, tuple(grid_shape), duration, courant_target=courant_target,
                           limiter=limiter, output_times=list(snap_times), on_output=on_output)
    # snapshots were written in reverse order, so ring index k has label t_final - t_rev
    n_out = len(labels)
    ring = ring[len(ring) - n_out:]
    times = np.sort(window.t_final - np.array(labels))
    wet = patch.aux.wet[spec.interior_slices()].copy() if hasattr(patch.aux, "wet") else None
    store = AdjointSnapshotStore.from_device(times, ring, origin, wx, wy, window, wet)
    if not keep_on_device:
        store.fields = [UniformField(values=ring[k].cpu().numpy(), origin=origin, dx=wx, dy=wy,
                                     time=float(times[k])) for k in range(n_out)]
    return store


class AdjointFlagging:
    """Flagging strategy backed by the snapshot ring (adjoint.py:260-277)."""

    name = "adjoint"

    def __init__(self, store: AdjointSnapshotStore, window: TimeWindow, tolerance: float,
                 time_interp: bool = False):
        if store is None:
            raise ConfigurationError("adjoint strategy configured without a store")
        if tolerance <= 0:
            raise ValueError("tolerance must be positive")
        self.store = store
        self.window = window
        self.tolerance = tolerance
        self.time_interp = time_interp

    def evaluate(self, patch):
        flags, _, _ = flag_level([patch], patch.time, self.store, self.window, self.tolerance,
                                 time_interp=self.time_interp)
        return flags[0]

    def evaluate_level_bits(self, patches):
        """One K3 launch -> (packed flag words on the device, level store)."""
        return flag_level(patches, patches[0].time, self.store, self.window, self.tolerance,
                          time_interp=self.time_interp, device_bits=True)

    def evaluate_level(self, patches):
        """All patches of a level in one K3 launch -> (flags list, raw counts)."""
        t = patches[0].time
        flags, counts, _ = flag_level(patches, t, self.store, self.window, self.tolerance,
                                      time_interp=self.time_interp)
        return flags, counts
