"""Single-patch stepping API on the device (drop-in for the reference's solver.py).

Every function keeps the reference signature and error behaviour
(/root/reference/pkg/src/adjamr/solver.py) but runs the hand-written sm_100a
kernels through the C ABI: K1 (step), K2 (ghost fill).  Material sampling
from user callables and dt selection stay on the host.
"""
from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np

from . import _lib, device
from .equations import EquationSet
from .geometry import Patch, PatchHierarchy

LIMITERS = ("none", "minmod", "MC", "superbee")
DEFAULT_VARIANT = _lib.VARIANT_FAST


class CflViolationError(RuntimeError):
    """A step exceeded the unit Courant number and was rejected (solver.py:23)."""


class NumericalBlowupError(RuntimeError):
    """A step produced NaN or Inf (solver.py:27)."""


class SchedulingError(RuntimeError):
    """Coarse data does not bracket the requested interpolation time (solver.py:31)."""


@dataclass(frozen=True)
class BoundarySpec:
    """Physical boundary condition per side: 'wall' or 'outflow' (solver.py:35-56).
    Extension: 'periodic' on both sides of an axis (BASELINE C3's periodic x;
    the reference has no periodic condition), for levels whose patches span
    that axis."""

    left: str = "wall"
    right: str = "wall"
    bottom: str = "wall"
    top: str = "wall"

    def __post_init__(self):
        for side in (self.left, self.right, self.bottom, self.top):
            if side not in ("wall", "outflow", "periodic"):
                raise ValueError(f"unknown boundary condition {side!r}")
        if (self.left == "periodic") != (self.right == "periodic") or \
                (self.bottom == "periodic") != (self.top == "periodic"):
            raise ValueError("periodic boundaries come in pairs (both sides of an axis)")

    def side(self, axis: int, high: bool) -> str:
        if axis == 0:
            return self.right if high else self.left
        return self.top if high else self.bottom


class StepResult:
    """Result of step_patch (solver.py:59-62).  ``state`` is fetched from the
    device lazily, so callers that ignore it pay no device-to-host copy."""

    def __init__(self, state, max_courant: float):
        self._state = state
        self.max_courant = max_courant

    @property
    def state(self) -> np.ndarray:
        return self._state() if callable(self._state) else self._state


# ---------------------------------------------------------------------------
# materials (host: arbitrary Python callables), solver.py:149-205


def _fix_aux_ghosts(arr: np.ndarray, axis: int, high: bool, g: int, wall, periodic: bool = False):
    n = arr.shape[axis]
    idx = [slice(None)] * arr.ndim
    src = [slice(None)] * arr.ndim
    if high:
        idx[axis] = slice(n - g, n)
        src[axis] = (slice(g, 2 * g) if periodic else
                     slice(n - g - 1, n - 2 * g - 1, -1) if wall else slice(n - g - 1, n - g))
    else:
        idx[axis] = slice(0, g)
        src[axis] = (slice(n - 2 * g, n - g) if periodic else
                     slice(2 * g - 1, g - 1, -1) if wall else slice(g, g + 1))
    arr[tuple(idx)] = arr[tuple(src)]


_FIELDS: dict = {}


def _field_names(cls):
    names = _FIELDS.get(cls)
    if names is None:
        import dataclasses
        names = _FIELDS[cls] = tuple(f.name for f in dataclasses.fields(cls))
    return names


def sample_patch_material(patch: Patch, equation: EquationSet, boundary: BoundarySpec,
                          level_shape: tuple[int, ...]):
    """Sample the material at cell centres (incl. ghosts), then mirror (wall)
    or extrapolate (outflow) it into physical-boundary ghosts."""
    spec = patch.spec
    cs = spec.cell_centers(include_ghost=True)
    if spec.ndim == 1:
        mat = equation.sample_material(cs[0])
    else:
        xx, yy = np.meshgrid(cs[0], cs[1], indexing="ij")
        mat = equation.sample_material(xx, yy)
    names = _field_names(type(mat))
    arrays = {n: np.array(getattr(mat, n), copy=True) for n in names if isinstance(getattr(mat, n), np.ndarray)}
    g = spec.ghost_width
    for axis in range(spec.ndim):
        for high in (False, True):
            at_edge = spec.hi[axis] == level_shape[axis] - 1 if high else spec.lo[axis] == 0
            if at_edge:
                wall = boundary.side(axis, high) == "wall"
                per = boundary.side(axis, high) == "periodic"
                for arr in arrays.values():
                    _fix_aux_ghosts(arr, axis, high, g, wall, per)
    others = {n: getattr(mat, n) for n in names if n not in arrays}
    patch.aux = type(mat)(**arrays, **others)
    if patch._store is not None:
        patch._store._dry = None
        patch._store._static_speed = None
        patch._store.uniform_mat = device.LevelStore._uniform_material(patch._store.patches)
        for key in [k for k in patch._store._scratch if isinstance(k, tuple) and k[0] in ("job_uniform", "job_uniform_np", "tiles_edge_first")]:
            del patch._store._scratch[key]
        av = patch._store.aux_view(patch._slot)
        import torch
        for k, pl in enumerate(patch.aux.planes()):
            av[k].copy_(torch.from_numpy(np.ascontiguousarray(pl, dtype=float)))
    return patch.aux


def _finish_material(patch, mat_cls, arrays, others, boundary, level_shape):
    spec = patch.spec
    g = spec.ghost_width
    for axis in range(spec.ndim):
        for high in (False, True):
            at_edge = spec.hi[axis] == level_shape[axis] - 1 if high else spec.lo[axis] == 0
            if at_edge:
                wall = boundary.side(axis, high) == "wall"
                per = boundary.side(axis, high) == "periodic"
                for arr in arrays.values():
                    _fix_aux_ghosts(arr, axis, high, g, wall, per)
    patch.aux = mat_cls(**arrays, **others)


def _centres_flat(specs):
    """Ghost-inclusive cell centres of many patches of one level, flattened
    patch after patch in meshgrid 'ij' order: the values cell_centers()
    gives (origin + (index + 0.5) * width, the same operations), built
    without a per-patch meshgrid.  Returns (coordinate arrays, shapes)."""
    nd, g = specs[0].ndim, specs[0].ghost_width
    lo = np.array([s.lo for s in specs], dtype=np.int64).reshape(len(specs), nd) - g
    n = np.array([s.shape for s in specs], dtype=np.int64).reshape(len(specs), nd) + 2 * g
    o, w = specs[0].origin, specs[0].widths
    nx = n[:, 0]
    ri = np.arange(int(nx.sum()), dtype=np.int64) - np.repeat(np.cumsum(nx) - nx, nx)   # row within patch
    xrow = o[0] + ((np.repeat(lo[:, 0], nx) + ri) + 0.5) * w[0]
    shapes = [tuple(r) for r in n.tolist()]
    if nd == 1:
        return (xrow,), shapes
    rlen = np.repeat(n[:, 1], nx)                                                        # cells per row
    j = np.arange(int(rlen.sum()), dtype=np.int64) - np.repeat(np.cumsum(rlen) - rlen, rlen)
    y = o[1] + ((np.repeat(np.repeat(lo[:, 1], nx), rlen) + j) + 0.5) * w[1]
    return (np.repeat(xrow, rlen), y), shapes


def sample_patches_material(patches, equation: EquationSet, boundary: BoundarySpec, level_shape: tuple[int, ...]):
    """sample_patch_material for many new patches of one level.  The material
    model is called once on the concatenated (flattened) ghost-inclusive
    cell-centre coordinates of all patches; each patch's values are then
    those of its own call (verified exactly against a per-patch call on the
    first patch; any difference or error falls back to one call per patch).
    Each patch's material arrays are views into the one sampled array per
    field (disjoint slices; the physical-boundary ghost fixes write only
    their own patch's slice)."""
    P = len(patches)
    if P < 4 or any(p._store is not None for p in patches) or os.environ.get("ADJAMR_BATCH_MATERIAL") == "0":
        for p in patches:
            sample_patch_material(p, equation, boundary, level_shape)
        return
    specs = [p.spec for p in patches]
    nd = specs[0].ndim
    s0 = specs[0]
    same_geom = all(s.origin == s0.origin and s.dx == s0.dx and s.dy == s0.dy and s.ghost_width == s0.ghost_width
                    for s in specs)
    try:
        if not same_geom:
            raise ValueError("patches of different geometry")
        coords, shapes = _centres_flat(specs)
        sizes = [int(np.prod(sh)) for sh in shapes]
        mat = equation.sample_material(*coords)
        cs0 = s0.cell_centers(include_ghost=True)
        mat0 = (equation.sample_material(cs0[0]) if nd == 1 else
                equation.sample_material(*np.meshgrid(cs0[0], cs0[1], indexing="ij")))
        names = _field_names(type(mat))
        arr_names = [n for n in names if isinstance(getattr(mat0, n), np.ndarray)]
        ok = type(mat0) is type(mat) and all(
            isinstance(getattr(mat, n), np.ndarray) and getattr(mat, n).shape == (sum(sizes),)
            and np.array_equal(getattr(mat, n)[:sizes[0]].reshape(shapes[0]), getattr(mat0, n)) for n in arr_names)
        ok = ok and all(getattr(mat, n) == getattr(mat0, n) for n in names if n not in arr_names)
    except Exception:
        ok = False
    if not ok:
        for p in patches:
            sample_patch_material(p, equation, boundary, level_shape)
        return
    others = {n: getattr(mat, n) for n in names if n not in arr_names}
    fields = {n: np.array(getattr(mat, n), copy=True) for n in arr_names}   # owned, writable
    off = np.concatenate([[0], np.cumsum(sizes)]).tolist()
    mat_cls = type(mat)
    for k, p in enumerate(patches):
        _finish_material(p, mat_cls, {n: f[off[k]:off[k + 1]].reshape(shapes[k]) for n, f in fields.items()},
                         others, boundary, level_shape)


# ---------------------------------------------------------------------------
# store helpers


def store_of(patch: Patch) -> device.LevelStore:
    """The patch's level store (a private single-patch store if it has none)."""
    if patch._store is None:
        device.LevelStore([patch])
    return patch._store


def level_store(patches: list[Patch]) -> device.LevelStore:
    """One store holding exactly ``patches`` in order (re-homing if needed)."""
    st = patches[0]._store
    if st is not None and len(st.patches) == len(patches) and all(
            a is b and b._store is st for a, b in zip(st.patches, patches)):
        return st
    for p in patches:
        if p._store is not None:
            old = p.state_old if p._store.has_old(p._slot) else p._host_old
            _ = p.state                   # pull the authoritative state to the host
            p._host_old = None if old is None else np.array(old, copy=True)
            p._time, p._time_old = p.time, p.time_old
            p._loc_own = "host"
            p._store = None
    return device.LevelStore(patches)


def _cfl(smax: np.ndarray, dtdx: float, dtdy: float, ndim: int) -> np.ndarray:
    sx = smax[:, 0] * dtdx
    return sx if ndim == 1 else np.maximum(sx, smax[:, 1] * dtdy)


# ---------------------------------------------------------------------------
# K1


def step_patch(patch: Patch, dt: float, equation: EquationSet, limiter: str = "MC",
               variant: int | None = None) -> StepResult:
    """Advance one patch by dt on the device (solver.py:515-522).

    Raises CflViolationError before any mutation, NumericalBlowupError after
    the update, ValueError on bad arguments.
    """
    if dt <= 0:
        raise ValueError("dt must be positive")
    if limiter not in LIMITERS:
        raise ValueError(f"unknown limiter {limiter!r}")
    variant = DEFAULT_VARIANT if variant is None else variant
    st = store_of(patch)
    st.sync_in()
    st.fold_ghosts()
    busy = [st.cur] + ([st.old] if st.old is not None else [])
    out = st._free(*busy)
    if len(st.patches) == 1:
        smax, bad = device.launch_step(st, dt, equation, limiter, variant, out)
    else:
        smax, bad = _launch_single(st, patch._slot, dt, equation, limiter, variant, out)
    spec = patch.spec
    dtdx = dt / spec.dx
    dtdy = dt / spec.dy if spec.ndim == 2 else 0.0
    k = 0 if len(st.patches) == 1 else patch._slot
    sm = smax.cpu().numpy()
    nonfinite = bool(bad[k].item())
    cfl = float(_cfl(sm[k:k + 1], dtdx, dtdy, spec.ndim)[0])
    if cfl > 1.0 + 1e-12:
        raise CflViolationError(f"Courant number {cfl:.4f} > 1")
    if len(st.patches) == 1:
        st.ghost_src = st.cur
        st.cur = out
    else:
        st._unalias()
        g = st.g
        src = st._view(st.buf[out], patch._slot, st.m)
        dst = st.view(patch._slot)
        if spec.ndim == 2:
            dst[:, g:-g, g:-g].copy_(src[:, g:-g, g:-g])
        else:
            dst[:, g:-g].copy_(src[:, g:-g])
    patch._loc = "device"
    patch.time += dt
    if nonfinite:
        raise NumericalBlowupError(f"non-finite state at t={patch.time}")
    return StepResult(lambda: patch.state, cfl)


def step_patch_host(patch: Patch, host_state, dt: float, equation: EquationSet, boundary: BoundarySpec,
                    level_shape: tuple[int, ...], limiter: str = "MC", slabs: int | None = None,
                    wait: bool = True) -> StepResult:
    """fill_ghost_physical + step_patch (solver.py:125-146, 515-522) on a state
    that lives in host memory, as the reference keeps it: ``host_state``
    (m, nx+2g, ny+2g) -- a torch CPU tensor, pinned for full overlap -- is
    read, advanced by dt and overwritten in place; the patch's device copy
    holds the same state afterwards.  Row slabs stream through the device
    with the host-to-device copy, the step and the device-to-host copy of
    consecutive slabs overlapping.  Needs the fast 2D path (static CFL bound);
    raises CflViolationError before any mutation.

    ``wait=False``: return with the device-to-host copies in flight, like a
    ``non_blocking`` torch copy.  The next call (same host buffer) overlaps its
    host-to-device copies with them slab by slab; ``host_stream_finish``
    completes them and raises NumericalBlowupError for any non-finite step."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    if limiter not in LIMITERS:
        raise ValueError(f"unknown limiter {limiter!r}")
    st = store_of(patch)
    if len(st.patches) != 1 or not device.fast_static(st, equation, _lib.VARIANT_FAST):
        raise ValueError("step_patch_host needs a single 2D patch store on the static-CFL fast path")
    spec = patch.spec
    dtdx, dtdy = dt / spec.dx, dt / spec.dy
    cfl = float(_cfl(st.static_speed_np(), dtdx, dtdy, 2)[0])
    if cfl > 1.0 + 1e-12:
        raise CflViolationError(f"Courant number {cfl:.4f} > 1")
    if slabs is None:      # measured on C4: 8 slabs (4-8 within box-to-box spread for chained steps)
        slabs = 8
    bad = device.stream_step(st, host_state, dt, equation, boundary, level_shape, limiter, slabs, wait=wait)
    patch._loc = "device"
    patch.time += dt
    if bad:
        raise NumericalBlowupError(f"non-finite state at t={patch.time}")
    return StepResult(lambda: patch.state, cfl)


def host_stream_finish(patch: Patch):
    """Completes the host state of ``step_patch_host(..., wait=False)`` calls."""
    if device.stream_finish(store_of(patch)):
        raise NumericalBlowupError(f"non-finite state at or before t={patch.time}")


def _launch_single(st, slot, dt, equation, limiter, variant, out):
    """Step one patch of a multi-patch store (work tables restricted to it)."""
    if variant == _lib.VARIANT_FAST and st.any_dry() and not device.fast_dry_ok(st, equation):
        variant = _lib.VARIANT_EXACT
    key = ("single", variant, slot)
    if key not in st._tiles:
        tiles, ntile, jobs, njob = st.tiles(variant)
        allrows = np.frombuffer(tiles.cpu().numpy().tobytes(), dtype=_lib.TILE_DTYPE)[:ntile]
        if jobs is None:
            sub = allrows[allrows["patch"] == slot]
            st._tiles[key] = (device._dev_table(sub), len(sub), None, len(sub))
        else:
            offs = jobs.cpu().numpy()
            rows, new_offs = [], [0]
            for j in range(len(offs) - 1):
                seg = allrows[offs[j]:offs[j + 1]]
                seg = seg[seg["patch"] == slot]
                for r in seg:
                    r = r.copy()
                    r["pad"] = 0
                    rows.append(r)
                    new_offs.append(len(rows))
            arr = np.array(rows, dtype=_lib.TILE_DTYPE)
            st._tiles[key] = (device._dev_table(arr), len(arr),
                              device._torch().from_numpy(np.array(new_offs, dtype=np.int32)).to("cuda"), len(arr))
    saved = st._tiles[variant]
    st._tiles[variant] = st._tiles[key]
    try:
        return device.launch_step(st, dt, equation, limiter, variant, out)
    finally:
        st._tiles[variant] = saved


# ---------------------------------------------------------------------------
# K2 single-patch entry points


def fill_ghost_physical(patch: Patch, boundary: BoundarySpec, equation: EquationSet,
                        level_shape: tuple[int, ...]):
    """Wall / outflow ghosts of one patch (solver.py:125-146), on the device."""
    st = store_of(patch)
    if len(st.patches) == 1:
        device.fill_physical(st, boundary, equation, level_shape)
    else:
        from . import amr
        amr._fill_physical_subset(st, [patch._slot], boundary, equation, level_shape)


def fill_ghost_same_level(patch: Patch, level_patches: list[Patch]):
    """Copy overlapping same-level interiors into this patch's ghosts (solver.py:208-224)."""
    from . import amr
    amr.fill_same_level(level_patches, only=patch)


def fill_ghost_from_coarse(fine_patch: Patch, hierarchy: PatchHierarchy, t: float):
    """Space-time interpolated in-domain ghosts from the coarser level (solver.py:227-286)."""
    from . import amr
    if fine_patch.spec.level < 2:
        return
    amr.fill_from_coarse(hierarchy, fine_patch.spec.level, t, only=fine_patch)


# ---------------------------------------------------------------------------
# dt selection and the uniform loop (host control, device work)


def select_dt(hierarchy: PatchHierarchy, equation: EquationSet,
              courant_target: float = 0.9, dt_max: float = np.inf) -> float:
    """Coarse-level dt from the CFL target (solver.py:525-542)."""
    if not 0.0 < courant_target <= 1.0:
        raise ValueError("courant_target must be in (0, 1]")
    speed = 0.0
    for p in hierarchy.patches(1):
        sl = p.spec.interior_slices()
        speed = max(speed, float(np.max(equation.max_speed(p.aux[sl]), initial=0.0)))
    if speed == 0.0:
        return dt_max
    wx, wy = hierarchy.widths(1)
    dt = courant_target * wx / speed
    if hierarchy.ndim == 2:
        dt = min(dt, courant_target * wy / speed)
    return min(dt, dt_max)


def integrate_patch(patch: Patch, equation: EquationSet, boundary: BoundarySpec,
                    level_shape: tuple[int, ...], t_end: float, *,
                    courant_target: float = 0.9, limiter: str = "MC",
                    dt_max: float = np.inf, dt_fixed: float | None = None,
                    output_times=(), on_output=None, on_step=None, variant: int | None = None):
    """Advance one uniform patch to t_end (solver.py:545-586): K2 physical
    fill + K1 per step on the device, outputs hit exactly."""
    sl = patch.spec.interior_slices()
    speed = float(np.max(equation.max_speed(patch.aux[sl]), initial=0.0))
    if dt_fixed is not None:
        base = dt_fixed
    elif speed == 0.0:
        base = dt_max
    else:
        base = courant_target * patch.spec.dx / speed
        if patch.spec.ndim == 2:
            base = min(base, courant_target * patch.spec.dy / speed)
        base = min(base, dt_max)
    pending = sorted(output_times)
    eps = 1e-9 * max(abs(t_end), 1.0)

    def flush():
        while pending and pending[0] <= patch.time + eps:
            t_out = pending.pop(0)
            if on_output is not None:
                on_output(t_out, patch)

    flush()
    while patch.time < t_end - eps:
        dt = min(base, t_end - patch.time)
        if pending:
            dt = min(dt, pending[0] - patch.time)
        fill_ghost_physical(patch, boundary, equation, level_shape)
        step_patch(patch, dt, equation, limiter, variant=variant)
        if on_step is not None:
            on_step(patch)
        flush()


# advance_uniform: the physical ghost fill runs inside the step launch (ADJ_STEP_PHYS_IN) for a
# patch spanning its level; ADJAMR_PHYS_IN=0 launches fill_ghost_physical separately
USE_PHYS_IN = os.environ.get("ADJAMR_PHYS_IN", "1") != "0"


def advance_uniform(patch: Patch, equation: EquationSet, boundary: BoundarySpec,
                    level_shape: tuple[int, ...], dt: float, nsteps: int, limiter: str = "MC",
                    variant: int | None = None, stream=None, graph: bool = True) -> float:
    """nsteps fixed-dt steps of one uniform patch with physical boundaries,
    device-resident and without a host sync per step (the batched form of
    the integrate_patch loop, solver.py:578-586).  On the static-CFL fast
    path the Courant number is known on the host and the fill+step pair is
    replayed from a CUDA graph; non-finite values are accumulated on the
    device and raised after the batch.  Returns the maximum Courant number."""
    import torch
    variant = DEFAULT_VARIANT if variant is None else variant
    st = store_of(patch)
    st.sync_in(stream)
    spec = patch.spec
    dtdx = dt / spec.dx
    dtdy = dt / spec.dy if spec.ndim == 2 else 0.0
    static = device.fast_static(st, equation, variant)
    if static:
        cfl = float(_cfl(st.static_speed_np(), dtdx, dtdy, spec.ndim)[0])
        if cfl > 1.0 + 1e-12:
            raise CflViolationError(f"Courant number {cfl:.4f} > 1")

        # a patch spanning its level has only physical ghosts: the step launch fills them itself
        # (ADJ_STEP_PHYS_IN; each warp job the ones its strip reads), no fill launch in between
        pin = (USE_PHYS_IN and len(st.patches) == 1 and st.g == 2 and spec.ndim == 2 and min(spec.shape) >= 2
               and st.all_edges_physical(level_shape) and not st.two_rows())
        if pin and "periodic" in (boundary.left, boundary.right, boundary.bottom, boundary.top):
            device.check_periodic(st, boundary, level_shape)

        def one_step():
            if pin:
                st.prepare_write(full_ghosts=True, stream=stream)   # the launch writes every ghost cell
            else:
                device.fill_physical(st, boundary, equation, level_shape, stream)
            st.fold_ghosts(stream)
            out = st._free(*([st.cur] + ([st.old] if st.old is not None else [])))
            device.launch_step(st, dt, equation, limiter, variant, out, stream, accumulate=True,
                               phys_in=(boundary, equation, tuple(level_shape)) if pin else None)
            st.ghost_src = st.cur
            st.cur = out

        done = 0
        key = ("uniform_graph", dt, limiter, tuple(level_shape), boundary, id(equation))
        key1 = ("uniform_graph1",) + key[1:]

        def cached():
            return st._scratch.get(key + ((st.cur, st.old, st.ghost_src),)) if graph else None

        def capture_single():
            """Capture (without running) one step from the current buffer roles;
            the host roles advance as if it ran."""
            roles = (st.cur, st.old, st.ghost_src)
            cg1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg1):
                one_step()
            st._scratch[key1 + (roles,)] = (cg1, (st.cur, st.old, st.ghost_src))

        def single_step():
            """One step from the single-step graph of the current buffer roles
            (both parities are captured next to the pair)."""
            roles = (st.cur, st.old, st.ghost_src)
            e = st._scratch.get(key1 + (roles,))
            if e is None:
                torch.cuda.synchronize()
                capture_single()
                e = st._scratch[key1 + (roles,)]
            else:
                st.cur, st.old, st.ghost_src = e[1]
            e[0].replay()
            patch.time += dt

        captured = graph and any(isinstance(kk, tuple) and kk[:6] == key for kk in st._scratch)
        g = cached()
        if graph and g is None and captured and nsteps >= 1:
            single_step()                   # other parity of a captured pair: realign from a graph
            done += 1
            g = cached()
        if graph and (g is not None or nsteps - done >= 4):
            if g is None:
                for i in range(st.NBUF):
                    st._ensure_buf(i)
                one_step(); one_step()          # warm-up (no capture of first-touch work)
                done += 2
                patch.time += dt
                patch.time += dt
                roles = (st.cur, st.old, st.ghost_src)
                torch.cuda.synchronize()
                cg = torch.cuda.CUDAGraph()
                with torch.cuda.graph(cg):
                    one_step(); one_step()
                if (st.cur, st.old, st.ghost_src) != roles:
                    raise RuntimeError("uniform step pair is not 2-periodic")
                g = (cg, roles)
                st._scratch[key + (roles,)] = g
                capture_single()                # single steps of both parities (odd counts, realignment)
                capture_single()
                if (st.cur, st.old, st.ghost_src) != roles:
                    raise RuntimeError("uniform single steps are not 2-periodic")
                # the host state already reflects the captured pair; run it once
                cg.replay()
                done += 2
                patch.time += dt
                patch.time += dt
            while nsteps - done >= 2:
                g[0].replay()
                done += 2
                patch.time += dt
                patch.time += dt
        while done < nsteps:
            if g is not None:
                single_step()
            else:
                one_step()
                patch.time += dt
            done += 1
        patch._loc = "device"
        if st.nonfinite_acc is not None and bool(st.nonfinite_acc.any().item()):
            st.nonfinite_acc.zero_()
            raise NumericalBlowupError(f"non-finite state at t={patch.time}")
        return cfl
    track = torch.zeros(2, dtype=torch.float64, device="cuda")
    badacc = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(nsteps):
        device.fill_physical(st, boundary, equation, level_shape, stream)
        st.fold_ghosts(stream)
        busy = [st.cur] + ([st.old] if st.old is not None else [])
        out = st._free(*busy)
        smax, bad = device.launch_step(st, dt, equation, limiter, variant, out, stream)
        torch.maximum(track, smax.reshape(-1, 2).amax(0), out=track)
        badacc.bitwise_or_(bad.amax().reshape(1))
        st.ghost_src = st.cur
        st.cur = out
        patch.time += dt
    patch._loc = "device"
    sm = track.cpu().numpy()[None, :]
    cfl = float(_cfl(sm, dtdx, dtdy, spec.ndim)[0])
    if cfl > 1.0 + 1e-12:
        raise CflViolationError(f"Courant number {cfl:.4f} > 1")
    if int(badacc.item()):
        raise NumericalBlowupError(f"non-finite state at t={patch.time}")
    return cfl
