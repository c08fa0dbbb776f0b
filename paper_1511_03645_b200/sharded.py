"""A uniform level sharded across ranks.

One process per GPU.  The level's x-rows (the slow, non-contiguous axis of
the patch box, ``Patch.state`` layout ``(m, nx+2g, ny+2g)``) are split into
contiguous slabs, one patch per rank.  Each step is the reference's uniform
loop (``integrate_patch``, solver.py:578-586: ``fill_ghost_physical`` then
``step_patch``) with one exchange in between: the g interior rows next to an
internal slab boundary go to the neighbouring rank and its g rows come back
into this patch's ghost rows.  Rows are sent whole (including their y ghost
columns, already filled by the neighbour's physical fill), so every rank's
ghost-inclusive box equals the corresponding window of the unsharded box
after ``fill_ghost_physical``.  The stepped interiors are bitwise identical
with the EXACT K1 variant; the FAST variant agrees to its 1e-12 tolerance
(its three register-ring column bodies are compiled separately, so where a
slab boundary shifts the march phase a cell may round differently).

The exchange is the path's only collective: point-to-point over
``torch.distributed`` (NCCL send/recv between GPUs over NVLink; gloo on CPU
tensors in the tests).  The CFL bound is static (``select_dt`` over the
global level = a MAX all-reduce of the per-slab material speed, once) and the
non-finite flag is reduced once per batch of steps, so no per-step
reduction is needed.  ``LocalTransport`` runs several shards in one process
(in-order copies), which the single-GPU tests use.
"""
from __future__ import annotations

import numpy as np


def slab_bounds(nx: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [x0, x1) of rank's slab: contiguous, balanced to within one row."""
    if not 0 <= rank < world or nx < world:
        raise ValueError("need 0 <= rank < world <= nx")
    base, extra = divmod(nx, world)
    x0 = rank * base + min(rank, extra)
    return x0, x0 + base + (1 if rank < extra else 0)


def halo_rows(q, m: int, plane: int, offset: int, pitch: int, r0: int, r1: int):
    """View (m, (r1-r0)*pitch) of box rows [r0, r1) of the patch at ``offset``
    in a level buffer of m component planes (1-D tensor of m*plane)."""
    return q.view(m, plane)[:, offset + r0 * pitch: offset + r1 * pitch]


class DistTransport:
    """Exchange with the x-neighbours through torch.distributed point-to-point."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def exchange(self, lo_send, hi_send):
        """lo_send -> rank-1, hi_send -> rank+1; returns (from rank-1, from rank+1).
        With a gloo group, device tensors are staged through host memory."""
        import torch
        import torch.distributed as dist
        t = lo_send if lo_send is not None else hi_send
        if t is not None and t.is_cuda and dist.get_backend(self.group) == "gloo":
            lo, hi = self.exchange(lo_send.cpu() if lo_send is not None else None,
                                   hi_send.cpu() if hi_send is not None else None)
            return (lo.to(t.device) if lo is not None else None, hi.to(t.device) if hi is not None else None)
        ops, lo_recv, hi_recv = [], None, None
        if self.rank > 0 and lo_send is not None:
            lo_recv = torch.empty_like(lo_send)
            ops += [dist.P2POp(dist.isend, lo_send, self.rank - 1, self.group),
                    dist.P2POp(dist.irecv, lo_recv, self.rank - 1, self.group)]
        if self.rank < self.world - 1 and hi_send is not None:
            hi_recv = torch.empty_like(hi_send)
            ops += [dist.P2POp(dist.isend, hi_send, self.rank + 1, self.group),
                    dist.P2POp(dist.irecv, hi_recv, self.rank + 1, self.group)]
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        return lo_recv, hi_recv

    def exchange_into(self, lo_send, hi_send, lo_recv, hi_recv):
        """exchange() into preallocated receive buffers (the graphed step's)."""
        lo, hi = self.exchange(lo_send, hi_send)
        if lo is not None:
            lo_recv.copy_(lo)
        if hi is not None:
            hi_recv.copy_(hi)


def exchange_x_halos(q, m: int, plane: int, offset: int, pitch: int, nx: int, g: int, transport,
                     has_lo: bool, has_hi: bool) -> None:
    """Send the g interior rows at each internal slab boundary and receive the
    neighbour's into the ghost rows (box rows [0, g) and [nx+g, nx+2g))."""
    lo = halo_rows(q, m, plane, offset, pitch, g, 2 * g).contiguous() if has_lo else None
    hi = halo_rows(q, m, plane, offset, pitch, nx, nx + g).contiguous() if has_hi else None
    lo_recv, hi_recv = transport.exchange(lo, hi)
    if has_lo:
        halo_rows(q, m, plane, offset, pitch, 0, g).copy_(lo_recv)
    if has_hi:
        halo_rows(q, m, plane, offset, pitch, nx + g, nx + 2 * g).copy_(hi_recv)


class LocalTransport:
    """Shards of one process (a list ordered by rank): exchange() of shard k
    hands back shard k-1's last rows and shard k+1's first rows, which
    ``exchange_local`` stages before any ghost row is overwritten."""

    def __init__(self, staged_lo, staged_hi):
        self.staged_lo, self.staged_hi = staged_lo, staged_hi

    def exchange(self, lo_send, hi_send):
        return self.staged_lo, self.staged_hi


def shard_patch(hierarchy, rank: int, world: int, nvar: int, level: int = 1):
    """The Patch covering rank's slab of a single-patch uniform level."""
    from .geometry import Patch
    shape = hierarchy.level_shape(level)
    x0, x1 = slab_bounds(shape[0], world, rank)
    hi = (x1 - 1,) + tuple(n - 1 for n in shape[1:])
    return Patch(hierarchy.make_spec(level, (x0,) + (0,) * (len(shape) - 1), hi), nvar)


def _layout(patch):
    from .solver import store_of
    st = store_of(patch)
    if len(st.patches) != 1:
        raise ValueError("a shard patch must own its store")
    t = st.table_np[0]
    return st, int(t["offset"]), int(t["pitch"])


def _edges(patch, level_shape):
    return patch.spec.lo[0] > 0, patch.spec.hi[0] < level_shape[0] - 1


def global_dt(hierarchy, equation, courant: float = 0.9, group=None) -> float:
    """select_dt (solver.py:525-542) over the union of every rank's level-1
    patches: the per-rank material speed maximum is MAX-all-reduced."""
    import torch
    import torch.distributed as dist
    speed = 0.0
    for p in hierarchy.patches(1):
        sl = p.spec.interior_slices()
        speed = max(speed, float(np.max(equation.max_speed(p.aux[sl]), initial=0.0)))
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor([speed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        speed = float(t.item())
    if speed == 0.0:
        return np.inf
    wx, wy = hierarchy.widths(1)
    dt = courant * wx / speed
    return min(dt, courant * wy / speed) if hierarchy.ndim == 2 else dt


def _step_one(patch, equation, boundary, level_shape, dt, limiter, variant, transport, stream):
    from . import device
    st, offset, pitch = _layout(patch)
    device.fill_physical(st, boundary, equation, level_shape, stream)
    st.fold_ghosts(stream)
    has_lo, has_hi = _edges(patch, level_shape)
    if (has_lo or has_hi) and not device.SHADOW:
        exchange_x_halos(st.buf[st.cur], st.m, st.plane, offset, pitch, patch.spec.shape[0], st.g, transport,
                         has_lo, has_hi)
    _launch(st, dt, equation, limiter, variant, stream)
    patch.time += dt


def _launch(st, dt, equation, limiter, variant, stream):
    """K1 into a free buffer; non-finite flags accumulate on the device
    (the EXACT kernel zeroes its per-launch flags, so they are OR-ed into a
    per-store accumulator)."""
    from . import _lib, device
    out = st._free(*([st.cur] + ([st.old] if st.old is not None else [])))
    _, bad = device.launch_step(st, dt, equation, limiter, variant, out, stream, accumulate=True)
    if variant != _lib.VARIANT_FAST and not device.SHADOW:
        acc = st.__dict__.get("_shard_bad")
        if acc is None:
            acc = st._shard_bad = bad.clone()
        else:
            acc.bitwise_or_(bad)
    st.ghost_src = st.cur
    st.cur = out


def _pending_bad(st):
    """Device int32 (1,) tensor: any non-finite value since the last check (then cleared)."""
    import torch
    flags = [t for t in (st.nonfinite_acc, st.__dict__.get("_shard_bad")) if t is not None]
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    for t in flags:
        out |= t.any().to(torch.int32).reshape(1)
        t.zero_()
    return out


def _usable(st, variant):
    from . import _lib
    if st.ndim != 2 or st.any_dry() or variant not in (_lib.VARIANT_FAST, _lib.VARIANT_EXACT):
        raise ValueError("sharded stepping needs a 2D level without dry cells (static CFL bound)")


def _check(st, dtdx, dtdy, ndim):
    from .solver import CflViolationError, _cfl
    cfl = float(_cfl(st.static_speed_np(), dtdx, dtdy, ndim)[0])
    if cfl > 1.0 + 1e-12:
        raise CflViolationError(f"Courant number {cfl:.4f} > 1")
    return cfl


def _split_tiles(st, nx, g):
    """FAST strip tables of the slab split into strips whose footprint
    (x +- g) stays inside the slab's interior rows (interior) and the rest
    (boundary, which read the exchanged ghost rows).  None if either is empty."""
    import numpy as np
    from . import _lib
    if st.two_rows():
        return None   # 64-row strips (ADJAMR_K1_ROWS=2) have no job table; the split would repack them
    key = ("shard_tiles", nx, g)
    hit = st._scratch.get(key)
    if hit is not None:
        return hit
    tiles, ntile, jobs, njob = st.tiles(_lib.VARIANT_FAST)
    rows = np.frombuffer(tiles.cpu().numpy().tobytes(), dtype=_lib.TILE_DTYPE)[:ntile].copy()
    offs = jobs.cpu().numpy() if jobs is not None else np.arange(ntile + 1, dtype=np.int32)
    touch = (rows["i0"] < g) | (rows["i0"] + rows["ni"] + g > nx)
    parts = []
    for want in (False, True):
        sel_rows, sel_offs = [], [0]
        for j in range(len(offs) - 1):
            seg = rows[offs[j]:offs[j + 1]]
            if bool(np.any(touch[offs[j]:offs[j + 1]])) == want:
                sel_rows.extend(seg)
                sel_offs.append(len(sel_rows))
        if not sel_rows:
            st._scratch[key] = None
            return None
        arr = np.array(sel_rows, dtype=_lib.TILE_DTYPE)
        parts.append((device_table(arr), len(arr), _torch_i32(sel_offs), len(sel_offs) - 1))
    st._scratch[key] = tuple(parts)
    return st._scratch[key]


def device_table(arr):
    from . import device
    return device._dev_table(arr)


def _torch_i32(vals):
    import numpy as np
    import torch
    return torch.from_numpy(np.array(vals, dtype=np.int32)).to("cuda")


def _launch_tiles(st, dt, equation, limiter, variant, out, tab):
    """K1 of the slab over one tile table (interior or boundary strips)."""
    from . import device
    saved = st._tiles[variant]
    st._tiles[variant] = tab
    try:
        device.launch_step(st, dt, equation, limiter, variant, out, None, accumulate=True)
    finally:
        st._tiles[variant] = saved


def _graphed_pair(patch, equation, boundary, level_shape, dt, limiter, variant, key):
    """Capture two consecutive steps of the slab as CUDA graphs around the
    (uncaptured) exchange.  Per step: pre = physical fill + ghost fold +
    packing of the boundary rows into persistent send buffers; FAST with an
    internal boundary: mid = K1 over the strips that do not read the ghost
    rows (it runs while the exchange is in flight on a side stream), post =
    unpacking into the ghost rows + K1 over the remaining strips; otherwise
    post = unpacking + K1 over the whole slab.  The buffer roles are
    2-periodic, as in advance_uniform."""
    import torch
    from . import _lib, device
    st, offset, pitch = _layout(patch)
    g, m, nx = st.g, st.m, patch.spec.shape[0]
    has_lo, has_hi = _edges(patch, level_shape)
    split = _split_tiles(st, nx, g) if (has_lo or has_hi) and variant == _lib.VARIANT_FAST else None
    bufs = [torch.empty((m, g * pitch), dtype=torch.float64, device="cuda") for _ in range(4)]
    send_lo, send_hi, recv_lo, recv_hi = bufs
    roles = (st.cur, st.old, st.ghost_src)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graphs = []
    with torch.cuda.stream(side):
        for _ in range(2):
            pre, mid, post = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(pre, stream=side):
                device.fill_physical(st, boundary, equation, level_shape)
                st.fold_ghosts()
                q = st.buf[st.cur]
                if has_lo:
                    send_lo.copy_(halo_rows(q, m, st.plane, offset, pitch, g, 2 * g))
                if has_hi:
                    send_hi.copy_(halo_rows(q, m, st.plane, offset, pitch, nx, nx + g))
            out = st._free(*([st.cur] + ([st.old] if st.old is not None else [])))
            if split is not None:
                with torch.cuda.graph(mid, stream=side):
                    _launch_tiles(st, dt, equation, limiter, variant, out, split[0])
            with torch.cuda.graph(post, stream=side):
                q = st.buf[st.cur]
                if has_lo:
                    halo_rows(q, m, st.plane, offset, pitch, 0, g).copy_(recv_lo)
                if has_hi:
                    halo_rows(q, m, st.plane, offset, pitch, nx + g, nx + 2 * g).copy_(recv_hi)
                if split is not None:
                    _launch_tiles(st, dt, equation, limiter, variant, out, split[1])
                else:
                    _launch(st, dt, equation, limiter, variant, None)
            if split is not None:
                st.ghost_src = st.cur
                st.cur = out
            graphs.append((pre, mid if split is not None else None, post))
    torch.cuda.current_stream().wait_stream(side)
    if (st.cur, st.old, st.ghost_src) != roles:
        raise RuntimeError("sharded step pair is not 2-periodic")
    entry = (graphs, bufs, has_lo, has_hi)
    st._scratch[key + (roles,)] = entry
    return entry


def advance_sharded(patch, equation, boundary, level_shape, dt: float, nsteps: int, transport,
                    limiter: str = "MC", variant: int | None = None, stream=None, group=None,
                    graph: bool = True) -> float:
    """nsteps of rank's slab (``solver.advance_uniform`` with the halo
    exchange).  2D levels without dry cells (either K1 variant): the Courant
    number is the static material bound, known on the host; the non-finite
    flag is accumulated on the device and all-reduced once at the end so
    every rank raises together.  ``graph``: pairs of steps replay CUDA graphs
    around the (uncaptured) exchange, so per step the host issues two graph
    launches and the exchange.  Returns this slab's Courant number."""
    import torch.distributed as dist
    from .solver import DEFAULT_VARIANT, NumericalBlowupError
    variant = DEFAULT_VARIANT if variant is None else variant
    st, _, _ = _layout(patch)
    st.sync_in(stream)
    _usable(st, variant)
    spec = patch.spec
    cfl = _check(st, dt / spec.dx, dt / spec.dy, 2)
    graph = graph and stream is None and hasattr(transport, "exchange_into")
    key = ("shard_graph", dt, limiter, variant, tuple(level_shape), boundary, id(equation))
    done = 0

    def cached():
        return st._scratch.get(key + ((st.cur, st.old, st.ghost_src),))

    def eager():
        _step_one(patch, equation, boundary, level_shape, dt, limiter, variant, transport, stream)

    entry = cached() if graph else None
    if graph and entry is None and nsteps >= 3 and any(isinstance(k, tuple) and k[:7] == key for k in st._scratch):
        eager()                              # the other parity of a captured pair: realign
        done += 1
        entry = cached()
    if graph and entry is None and nsteps - done >= 4:
        for i in range(st.NBUF):
            st._ensure_buf(i)
        eager(); eager()                     # warm-up: first-touch allocations happen outside capture
        done += 2
        entry = _graphed_pair(patch, equation, boundary, level_shape, dt, limiter, variant, key)
    if entry is not None:
        import torch
        graphs, (send_lo, send_hi, recv_lo, recv_hi), has_lo, has_hi = entry
        main = torch.cuda.current_stream()
        comm = st.__dict__.get("_shard_comm")
        if comm is None:
            comm = st._shard_comm = (torch.cuda.Stream(), torch.cuda.Event(), torch.cuda.Event())
        cstream, packed, received = comm
        while nsteps - done >= 2:
            for pre, mid, post in graphs:
                pre.replay()
                if has_lo or has_hi:
                    # the exchange runs on a side stream while the interior strips step
                    packed.record(main)
                    cstream.wait_event(packed)
                    with torch.cuda.stream(cstream):
                        transport.exchange_into(send_lo if has_lo else None, send_hi if has_hi else None,
                                                recv_lo, recv_hi)
                        received.record(cstream)
                    if mid is not None:
                        mid.replay()
                    main.wait_event(received)
                post.replay()
                patch.time += dt
            done += 2
    while done < nsteps:
        eager()
        done += 1
    patch._loc = "device"
    bad = _pending_bad(st)
    if isinstance(transport, DistTransport) and dist.is_initialized() and dist.get_world_size() > 1:
        if dist.get_backend(group) == "gloo":
            bad = bad.cpu()
        dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=group)
    if int(bad.item()):
        raise NumericalBlowupError(f"non-finite state at t={patch.time}")
    return cfl


def advance_local_shards(patches, equation, boundary, level_shape, dt: float, nsteps: int,
                         limiter: str = "MC", variant: int | None = None, stream=None) -> float:
    """Several slabs of one level in one process (ordered by x): each step
    fills every slab's physical ghosts, stages all internal-boundary rows,
    writes them into the neighbours' ghost rows, then steps every slab.  Same
    arithmetic as ``advance_sharded`` on separate ranks."""
    from . import device
    from .solver import DEFAULT_VARIANT, NumericalBlowupError
    variant = DEFAULT_VARIANT if variant is None else variant
    cfl = 0.0
    for p in patches:
        st, _, _ = _layout(p)
        st.sync_in(stream)
        _usable(st, variant)
        cfl = max(cfl, _check(st, dt / p.spec.dx, dt / p.spec.dy, 2))
    for _ in range(nsteps):
        lays = []
        for p in patches:
            st, offset, pitch = _layout(p)
            device.fill_physical(st, boundary, equation, level_shape, stream)
            st.fold_ghosts(stream)
            lays.append((st, offset, pitch, p.spec.shape[0]))
        g = lays[0][0].g
        firsts = [halo_rows(st.buf[st.cur], st.m, st.plane, o, pt, g, 2 * g).clone() for st, o, pt, nx in lays]
        lasts = [halo_rows(st.buf[st.cur], st.m, st.plane, o, pt, nx, nx + g).clone() for st, o, pt, nx in lays]
        for k, (p, (st, o, pt, nx)) in enumerate(zip(patches, lays)):
            has_lo, has_hi = _edges(p, level_shape)
            tr = LocalTransport(lasts[k - 1] if has_lo else None, firsts[k + 1] if has_hi else None)
            exchange_x_halos(st.buf[st.cur], st.m, st.plane, o, pt, nx, g, tr, has_lo, has_hi)
        for p in patches:
            st, _, _ = _layout(p)
            _launch(st, dt, equation, limiter, variant, stream)
            p.time += dt
    for p in patches:
        st, _, _ = _layout(p)
        p._loc = "device"
        if int(_pending_bad(st).item()):
            raise NumericalBlowupError(f"non-finite state at t={p.time}")
    return cfl
