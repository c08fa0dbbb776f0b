"""Per-level patch store in HBM and the launch wrappers of the C ABI.

Layout (include/adjamr_b200.h): every patch of a level occupies a
ghost-inclusive box of (nx+2g) rows by ``pitch`` elements (y contiguous,
pitch padded to a multiple of 4 so rows are 32 B aligned) inside one flat
plane; the m state components and the aux materials are separate planes
(structure of arrays).  Three state buffers rotate:

  cur        the current state,
  old        the state saved by save_old (reference ``Patch.state_old``),
  ghost_src  the buffer holding the current ghost values (after a step the
             new interior is in ``cur`` while the ghosts the reference would
             still hold are in the pre-step buffer; they are folded back with
             a ring copy before anything reads ``cur``'s ghosts).

A step reads ``cur`` and writes a free buffer, which replaces the reference's
``save_old`` full copy (geometry.py:123) and makes "raise before mutate" on a
CFL violation (solver.py:461) free: the new buffer is simply discarded.
"""
from __future__ import annotations

import os

import numpy as np

from . import _lib

_SLACK = 64   # elements of slack after each plane set (strip loads may over-read)

# Shadow mode: the host bookkeeping of a level sweep runs (buffer rotation,
# times, counters) but no work is launched -- used to keep the host state in
# step with CUDA-graph replays of the same sweep (amr.SweepGraph).
SHADOW = False
# wet/dry levels: per-job classes (all-wet jobs march without the wet/dry selects, all-dry jobs
# copy); ADJAMR_JOB_CLASS=0 runs every job through the wet/dry march
USE_JOB_CLASS = os.environ.get("ADJAMR_JOB_CLASS", "1") != "0"


class ParamSlots:
    """Per-launch scalar parameters of a captured sweep that change between
    replays (the coarse-to-fine time weight).  During capture every
    coarse-rect launch takes the next slot and reads its weight from device
    memory; shadow runs rewrite the host copy in the same order; ``upload``
    refreshes the device copy before a replay."""

    def __init__(self, cap=1024):
        import torch
        self.cap = cap
        self.vals: list[float] = []
        self.dev = torch.zeros(cap, dtype=torch.float64, device="cuda")

    def take(self, w: float) -> int:
        k = len(self.vals)
        if k >= self.cap:
            raise RuntimeError("too many time-weight slots in one captured sweep")
        self.vals.append(float(w))
        return int(self.dev.data_ptr()) + 8 * k

    def upload(self):
        """Stream-ordered copy of the slot values (a fresh pinned staging
        buffer per upload; torch keeps it alive until the copy ran)."""
        import torch
        if self.vals:
            h = torch.tensor(self.vals, dtype=torch.float64).pin_memory()
            self.dev[: len(self.vals)].copy_(h, non_blocking=True)

    def rewind(self):
        self.vals = []


PARAMS: ParamSlots | None = None


def _torch():
    import torch
    return torch


def _dev_table(arr: np.ndarray):
    """Upload a numpy structured table to the device as raw bytes."""
    torch = _torch()
    raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    if raw.size == 0:
        raw = np.zeros(8, np.uint8)
    return torch.from_numpy(raw.copy()).to("cuda", non_blocking=False)


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


# K1's homogeneous-material instantiation on levels whose aux planes are constant (False: always
# read the planes; same results bitwise)
USE_UNIFORM_MAT = os.environ.get("ADJAMR_UNIFORM_MAT", "1") == "1"
USE_MIXED_FIRST = os.environ.get("ADJAMR_MIXED_FIRST", "1") == "1"   # per-cell jobs at the head of the queue


class LevelStore:
    """All patches of one refinement level, resident in HBM."""

    NBUF = 3

    def __init__(self, patches):
        if not patches:
            raise ValueError("LevelStore needs at least one patch")
        torch = _torch()
        _lib.lib()   # fail loudly without the CUDA path
        self.patches = list(patches)
        if patches[0].aux is None:
            raise ValueError("patch has no material (call sample_patch_material first)")
        self.swe = hasattr(patches[0].aux, "wet")
        specs = [p.spec for p in patches]
        self.ndim = specs[0].ndim
        self.g = specs[0].ghost_width
        if any(s.ghost_width != self.g or s.ndim != self.ndim for s in specs):
            raise ValueError("patches of one store must share ghost width and dimension")
        self.m = patches[0].num_components
        self.naux = len(patches[0].aux.planes())
        # patch table, vectorised: boxes of nx+2g rows x pitch, each 32-element aligned
        nd, g = self.ndim, self.g
        lo = np.array([s.lo for s in specs], dtype=np.int64).reshape(len(specs), nd)
        shp = np.array([s.shape for s in specs], dtype=np.int64).reshape(len(specs), nd)
        nx = shp[:, 0]
        ny = shp[:, 1] if nd == 2 else np.ones_like(nx)
        NXa = nx + 2 * g
        NYa = ny + 2 * g if nd == 2 else np.ones_like(nx)
        pitch_a = (NYa + 3) // 4 * 4 if nd == 2 else np.ones_like(nx)
        size = (NXa * pitch_a + 31) // 32 * 32
        offs = np.cumsum(size) - size
        words = (nx * ny + 31) // 32
        fws = np.cumsum(words) - words
        tab = np.zeros(len(specs), dtype=_lib.PATCH_DTYPE)
        tab["offset"], tab["flag_word"], tab["nx"], tab["ny"], tab["pitch"] = offs, fws, nx, ny, pitch_a
        tab["lo_x"] = lo[:, 0]
        tab["lo_y"] = lo[:, 1] if nd == 2 else 0
        self.boxes = list(zip(offs.tolist(), NXa.tolist(), NYa.tolist(), pitch_a.tolist()))
        off = int(size.sum())
        fw = int(words.sum())
        self.plane = off + _SLACK
        self.flag_words = fw
        self.table_np = tab
        self.table = _dev_table(tab)
        self._edges_key = None
        self.buf = [torch.zeros(self.m * self.plane, dtype=torch.float64, device="cuda"), None, None]
        self.aux = torch.zeros(self.naux * self.plane, dtype=torch.float64, device="cuda")
        self.cur = 0
        self.old = None
        self.old_valid = np.zeros(len(specs), dtype=bool)
        self.ghost_src = 0
        self._tiles = {}
        self._scratch = {}
        self._dry = None
        self._static_speed = None
        self._static_speed_np = None
        self.all_device = False
        self.time_synced = False
        self.level_time = 0.0
        self.level_time_old = None
        self.total_cells = int((nx * ny).sum())
        self.max_ghost_cells = int((NXa * NYa - nx * ny).max())
        self._phys_args = {}
        self.nonfinite_acc = None
        # material planes of every patch assembled on the host, one upload
        host_aux = None
        if len({(b[1], b[2], b[3]) for b in self.boxes}) == 1:
            host_aux = np.zeros(self.naux * self.plane, dtype=np.float64)
            # one box shape (e.g. uniform 32^2 patches): one scatter for all patches
            _, NX0, NY0, P0 = self.boxes[0]
            stacked = np.stack([np.stack([np.asarray(pl, dtype=float).reshape(NX0, NY0) for pl in p.aux.planes()])
                                for p in patches])                          # (npatch, naux, NX, NY)
            cell = (np.arange(NX0)[:, None] * P0 + np.arange(NY0)[None, :]).reshape(-1)
            dst = (np.arange(self.naux)[None, :, None] * self.plane + offs[:, None, None] + cell[None, None, :])
            host_aux[dst.reshape(-1)] = stacked.reshape(-1)
            planes_all = (stacked[:, 0], stacked[:, 1]) if self.naux >= 2 else None
        if host_aux is not None:
            self.aux.copy_(torch.from_numpy(host_aux))
        else:
            # mixed box shapes: the planes of all patches concatenated on the host (one upload),
            # scattered into the boxes on the device (element e = ii * NY + jj of patch k goes to
            # offs[k] + ii * pitch[k] + jj)
            src = np.empty((self.naux, int((NXa * NYa).sum())), dtype=np.float64)
            planes = [p.aux.planes() for p in patches]
            for a in range(self.naux):
                np.concatenate([np.asarray(pl[a], dtype=float).reshape(-1) for pl in planes], out=src[a])
            planes_all = (src[0], src[1]) if self.naux >= 2 else None
            dev = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.int64)).to("cuda")
            nx_d, ny_d, off_d, pit_d = dev(NXa), dev(NYa), dev(offs), dev(pitch_a)
            nrow, ncell = int(NXa.sum()), src.shape[1]
            rep = lambda v, r, n: torch.repeat_interleave(v, r, output_size=n)   # no size sync
            ri = torch.arange(nrow, device="cuda") - rep(torch.cumsum(nx_d, 0) - nx_d, nx_d, nrow)
            rbase = rep(off_d, nx_d, nrow) + ri * rep(pit_d, nx_d, nrow)
            rlen = rep(ny_d, nx_d, nrow)
            j = torch.arange(ncell, device="cuda") - rep(torch.cumsum(rlen, 0) - rlen, rlen, ncell)
            dst = rep(rbase, rlen, ncell) + j
            self.aux.view(self.naux, self.plane)[:, dst] = torch.from_numpy(src).to("cuda")
        for k, p in enumerate(patches):
            self._attach(p, k, upload=False)
        # the assembled planes of all patches: one pass each instead of reductions per patch
        self.uniform_mat = None
        if USE_UNIFORM_MAT and not self.swe and self.ndim == 2 and planes_all is not None:
            self.uniform_mat = self._uniform_planes(*planes_all)

    @staticmethod
    def _uniform_planes(c, z):
        c0, z0 = float(c.flat[0]), float(z.flat[0])
        if not (np.isfinite(c0) and np.isfinite(z0) and c0 > 0.0 and z0 > 0.0):
            return None
        k = min(c.size, 4096)      # a varying medium usually shows in the first cells
        if not (np.all(c.flat[:k] == c0) and np.all(z.flat[:k] == z0)):
            return None
        return (c0, z0) if np.all(c == c0) and np.all(z == z0) else None

    @staticmethod
    def _uniform_material(patches):
        """(c, z) when every cell of every patch (ghosts included) has the same
        acoustic material, else None: K1's homogeneous-material instantiation
        (ADJ_STEP_UNIFORM_MAT) then computes the material terms once per strip."""
        if not USE_UNIFORM_MAT or hasattr(patches[0].aux, "wet") or patches[0].spec.ndim != 2:
            return None
        first = None
        for p in patches:
            c, z = p.aux.planes()[:2]
            u = LevelStore._uniform_planes(np.asarray(c), np.asarray(z))
            if u is None or (first is not None and u != first):
                return None
            first = u
        return first

    # ------------------------------------------------------------------ views
    def _view(self, t, slot, comps):
        off, NX, NY, pitch = self.boxes[slot]
        v = t.as_strided((comps, NX, NY), (self.plane, pitch, 1), off)
        return v if self.ndim == 2 else v[:, :, 0]

    def view(self, slot, which="cur"):
        idx = {"cur": self.cur, "old": self.old, "ghost": self.ghost_src}[which]
        return self._view(self.buf[idx], slot, self.m)

    def aux_view(self, slot):
        return self._view(self.aux, slot, self.naux)

    def _attach(self, patch, slot, upload=True):
        if patch.aux is None:
            raise ValueError("patch has no material (call sample_patch_material first)")
        if upload:
            av = self.aux_view(slot)
            for k, pl in enumerate(patch.aux.planes()):
                av[k].copy_(_torch().from_numpy(np.ascontiguousarray(pl, dtype=float)))
        patch._time = patch.time          # detach level-synchronised fields of a previous store
        patch._time_old = patch.time_old
        patch._loc_own = "host"           # uploaded by sync_in
        patch._store = self
        patch._slot = slot
        if patch._host_old is not None:
            self.old_valid[slot] = False

    # ------------------------------------------- level-synchronised fields
    def set_all_device(self):
        """Every patch's authoritative state is in cur (O(1))."""
        self.all_device = True

    def break_all_device(self):
        for p in self.patches:
            if p._store is self:
                p._loc_own = "device"
        self.all_device = False

    def set_level_times(self, t, t_old):
        """All patches share (time, time_old) (O(1))."""
        self.time_synced = True
        self.level_time = float(t)
        self.level_time_old = None if t_old is None else float(t_old)

    def break_time_sync(self):
        if not self.time_synced:
            return
        self.time_synced = False
        for p in self.patches:
            if p._store is self:
                p._time = self.level_time
                p._time_old = self.level_time_old

    # ------------------------------------------------------------ buffers
    def _ensure_buf(self, i):
        if self.buf[i] is None:
            torch = _torch()
            self.buf[i] = torch.zeros(self.m * self.plane, dtype=torch.float64, device="cuda")
        return self.buf[i]

    def settle_pending(self, stream=None):
        """Order the given (current) stream after the device-to-host copies of
        pending ``stream_step(wait=False)`` calls, which read this store's
        buffers: any other write to the store must not overtake them."""
        pend = self.__dict__.get("_stream_pending")
        if pend is not None:
            s = stream if stream is not None else _torch().cuda.current_stream()
            for ev in pend[1]:
                s.wait_event(ev)

    def _free(self, *busy, settle=True):
        if settle:
            self.settle_pending()
        for i in range(self.NBUF):
            if i not in busy:
                self._ensure_buf(i)
                return i
        raise RuntimeError("no free state buffer")

    def _unalias(self):
        """Make cur writable without touching the saved old buffer."""
        if self.old is not None and self.old == self.cur:
            nb = self._free(self.cur, self.ghost_src)
            if not SHADOW:
                self.buf[nb].copy_(self.buf[self.cur])
            if self.ghost_src == self.cur:
                self.ghost_src = nb
            self.cur = nb

    def fold_ghosts(self, stream=None):
        self.settle_pending(stream)
        """Copy the current ghost ring into cur (see module docstring)."""
        if self.ghost_src == self.cur:
            return
        self._unalias()
        if self.ghost_src != self.cur:
            ring_copy(self, self.buf[self.ghost_src], self.buf[self.cur], stream)
        self.ghost_src = self.cur

    def prepare_write(self, full_ghosts: bool = False, stream=None):
        """Before an in-place write to cur: unalias, and fold the ghosts unless
        the write rewrites every ghost cell."""
        self.settle_pending(stream)
        self._unalias()
        if full_ghosts:
            self.ghost_src = self.cur
        else:
            self.fold_ghosts(stream)

    # ----------------------------------------------------------- coherence
    def sync_in(self, stream=None):
        """Upload every patch whose authoritative state is on the host."""
        self.settle_pending(stream)
        if self.all_device:
            return
        pending = [p for p in self.patches if p._store is self and p._loc == "host"]
        if not pending:
            return
        self.prepare_write(stream=stream)
        torch = _torch()
        for p in pending:
            v = self.view(p._slot)
            v.copy_(torch.from_numpy(p._host), non_blocking=False)
            p._loc = "device"

    def download(self, slot, out: np.ndarray):
        self.settle_pending(None)
        torch = _torch()
        v = self.view(slot)
        if self.ghost_src != self.cur:
            full = self.view(slot, "ghost").clone()
            g = self.g
            if self.ndim == 2:
                full[:, g:-g, g:-g] = v[:, g:-g, g:-g]
            else:
                full[:, g:-g] = v[:, g:-g]
            v = full
        out[...] = v.cpu().numpy()
        del torch

    def has_old(self, slot) -> bool:
        return self.old is not None and bool(self.old_valid[slot])

    def download_old(self, slot, out: np.ndarray):
        self.settle_pending(None)
        out[...] = self.view(slot, "old").cpu().numpy()

    def drop_old(self, slot):
        self.old_valid[slot] = False

    def save_old(self, slot):
        """Per-patch save_old: copy the patch box into the old buffer."""
        self.sync_in()
        if self.old is None:
            self.old = self._free(self.cur, self.ghost_src)
            self.old_valid[:] = False
        if self.old != self.cur:
            self.fold_ghosts()
            self.view(slot, "old").copy_(self.view(slot))
        self.old_valid[slot] = True

    def save_old_all(self):
        """save_old for every patch of the level: alias, no copy."""
        self.sync_in()
        self.fold_ghosts()
        self.old = self.cur
        self.old_valid[:] = True

    # ------------------------------------------------------------- tables
    def edges_table(self, level_shape):
        """Patch table with edge bits for this level shape (all patches), and
        the compacted table of the patches that touch the domain boundary."""
        key = tuple(level_shape)
        if self._edges_key != key:
            tab = self.table_np.copy()
            for k, p in enumerate(self.patches):
                s = p.spec
                e = 0
                if s.lo[0] == 0:
                    e |= _lib.EDGE_XLO
                if s.hi[0] == level_shape[0] - 1:
                    e |= _lib.EDGE_XHI
                if self.ndim == 2:
                    if s.lo[1] == 0:
                        e |= _lib.EDGE_YLO
                    if s.hi[1] == level_shape[1] - 1:
                        e |= _lib.EDGE_YHI
                tab["edges"][k] = e
            self.table_np = tab
            self.table = _dev_table(tab)
            self._edges_key = key
            sel = tab[tab["edges"] != 0]
            self._edge_tab = (_dev_table(sel), len(sel))
        return self.table

    def all_edges_physical(self, level_shape) -> bool:
        full = 15 if self.ndim == 2 else 3
        self.edges_table(level_shape)
        return bool(np.all(self.table_np["edges"] == full))

    def _strip_length(self, ti_max, tj, warps_per_sm=12):
        """Strip march length: balance the last wave of the persistent warp
        queue against the 4 priming columns per strip.  A level that fits one
        wave of resident warps gets the shortest strips (a multiple of 4, for
        the fused restriction's alignment) that still fit it: all its jobs then
        run at once and fewer slots idle (C3 2048^2: 88-column strips, 1776
        jobs; measured with 86: K1 0.068 vs 0.075 ms with 96) -- or, better
        where possible, the shortest strips that fill two waves.  Across
        several waves the dynamic queue absorbs a partial last wave (C4:
        measured 128 best)."""
        torch = _torch()
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        slots = sms * warps_per_sm
        nxs = np.array([p.spec.shape[0] for p in self.patches], dtype=np.int64)
        nys = np.array([p.spec.shape[1] for p in self.patches], dtype=np.int64)
        rows = -(-nys // tj)

        def jobs(ti):
            return int(np.sum(-(-nxs // ti) * rows))
        force = os.environ.get("ADJAMR_K1_TI")
        if force:
            return int(force)
        best, best_score = ti_max, -1.0
        for ti in (ti_max, 112, 96, 80, 64, 48):
            if ti > ti_max:
                continue
            waves = jobs(ti) / slots
            score = (waves / np.ceil(waves)) * (ti / (ti + 4.0))
            if score > best_score + 1e-9:
                best, best_score = ti, score
        if jobs(ti_max) <= slots:
            one = next((ti for ti in range(16, ti_max + 1, 4) if jobs(ti) <= slots), None)
            if one is not None:
                score = (jobs(one) / slots) * (one / (one + 4.0))
                if score > best_score + 1e-9:
                    best = one
            # two full waves of strips of >= 32 columns, when the level allows them, beat the
            # single wave (C3 2048^2: 44-column strips, 3478 jobs: K1 0.067 vs 0.070 ms, and
            # 0.055 vs 0.063 ms with per-job materials, whose few per-cell jobs then no longer
            # set the duration of the one wave); levels of small patches have no such choice
            two = next((ti for ti in range(32, ti_max + 1, 4) if slots < jobs(ti) <= 2 * slots), None)
            if two is not None:
                best = two
        return best

    def two_rows(self) -> bool:
        """Use the two-rows-per-lane fast kernel (64-row strips; 2D, no dry
        cells) -- opt-in with ADJAMR_K1_ROWS=2: measured slower on B200 than
        the one-row kernel (255 registers with spills, 8 warps/SM)."""
        import os
        if self.ndim != 2 or self.any_dry():
            return False
        return os.environ.get("ADJAMR_K1_ROWS") == "2"

    def tiles(self, variant):
        """Work tables of a step variant: (tiles, ntile, job_offsets, njob).
        FAST 2D: strips of <= 28 rows x <= 128 columns; full strips are one warp
        job each, the short remainder strips of several patches are packed
        into shared warp jobs (lanes [pad, pad + nj + 4)), so 32-row patches
        keep 80% of the lanes busy instead of 50%."""
        if variant not in self._tiles:
            ni_t = _lib.C.c_int32()
            nj_t = _lib.C.c_int32()
            _lib.check(_lib.lib().adj_step_tile_shape(variant, self.ndim, _lib.C.byref(ni_t), _lib.C.byref(nj_t)),
                       "adj_step_tile_shape")
            ti, tj = ni_t.value, nj_t.value
            two = variant == _lib.VARIANT_FAST and self.two_rows()
            if two:
                tj = 60
            if variant == _lib.VARIANT_FAST and self.ndim == 2:
                ti = self._strip_length(ti, tj)
            full, short = [], {}
            for k, p in enumerate(self.patches):
                nx = p.spec.shape[0]
                ny = p.spec.shape[1] if self.ndim == 2 else 1
                for i0 in range(0, nx, ti):
                    ni = min(ti, nx - i0)
                    for j0 in range(0, ny, tj):
                        nj = min(tj, ny - j0)
                        if variant == _lib.VARIANT_FAST and self.ndim == 2 and not two and nj < tj and nj + 4 <= 16:
                            short.setdefault(ni, []).append((k, i0, j0, ni, nj, 0))
                        else:
                            full.append((k, i0, j0, ni, nj, 0))
            if two:
                full.sort(key=lambda r: (r[0], r[1], r[2]))
                arr = np.array(full, dtype=_lib.TILE_DTYPE)
                self._tiles[variant] = (_dev_table(arr), len(full), None, len(full))
            elif variant == _lib.VARIANT_FAST and self.ndim == 2:
                # x-segment major, then strips: concurrently running warps are
                # y-neighbours and share halo rows through L2
                full.sort(key=lambda r: (r[0], r[1], r[2]))
                rows, offs = list(full), list(range(len(full) + 1))
                for ni, lst in sorted(short.items()):
                    lane = 32
                    for (k, i0, j0, ni_, nj, _) in lst:
                        if lane + nj + 4 > 32:
                            lane = 0
                            offs.append(len(rows))
                        rows.append((k, i0, j0, ni_, nj, lane))
                        lane += nj + 4
                offs = sorted(set(offs + [len(rows)]))
                arr = np.array(rows, dtype=_lib.TILE_DTYPE)
                jobs = np.array(offs, dtype=np.int32)
                self._tiles[variant] = (_dev_table(arr), len(rows), _torch().from_numpy(jobs).to("cuda"),
                                        len(jobs) - 1)
            else:
                rows = full + [r for lst in short.values() for r in lst]
                arr = np.array(rows, dtype=_lib.TILE_DTYPE)
                self._tiles[variant] = (_dev_table(arr), len(rows), None, len(rows))
        return self._tiles[variant]

    def tiles_edge_first(self, level_shape):
        """The FAST job table with the jobs whose strips read physical ghost
        cells first (ADJ_STEP_PHYS_IN: those jobs fill them before they march,
        so they start early and the other warps' marches absorb the extra)."""
        key = ("tiles_edge_first", tuple(level_shape))
        hit = self._scratch.get(key)
        if hit is not None:
            return hit
        tiles, ntile, jobs, njob = self.tiles(_lib.VARIANT_FAST)
        rows = np.frombuffer(tiles.cpu().numpy().tobytes(), dtype=_lib.TILE_DTYPE)[:ntile].copy()
        offs = jobs.cpu().numpy().astype(np.int64) if jobs is not None else np.arange(ntile + 1, dtype=np.int64)
        nx = self.table_np["nx"][rows["patch"]]
        ny = self.table_np["ny"][rows["patch"]]
        edge = (rows["i0"] < 2) | (rows["i0"] + rows["ni"] + 2 > nx) | (rows["j0"] < 2) | (rows["j0"] + rows["nj"] + 2 > ny)
        job_edge = np.array([bool(edge[offs[j]:offs[j + 1]].any()) for j in range(len(offs) - 1)])
        # with per-job materials the few jobs that march per cell are the longest: they start first,
        # so none of them ends up in the tail of the last wave
        # (the same order by job class on a wet/dry level -- coastal, all-wet, all-dry -- measured
        # neutral on the C4 coastline, 0.2059 vs 0.2055 ms, and is not applied)
        prio = np.ones(len(job_edge), dtype=np.int64)
        if USE_MIXED_FIRST and self.job_uniform(tiles, ntile, jobs, njob) is not None:
            prio[self._scratch[("job_uniform_np", _ptr(tiles))][:, 0] == 0.0] = 0
        order = np.argsort(2 * prio + (~job_edge).astype(np.int64), kind="stable")
        new_rows, new_offs = [], [0]
        for j in order:
            new_rows.extend(rows[offs[j]:offs[j + 1]])
            new_offs.append(len(new_rows))
        arr = np.array(new_rows, dtype=_lib.TILE_DTYPE)
        hit = (_dev_table(arr), len(arr), _torch().from_numpy(np.array(new_offs, dtype=np.int32)).to("cuda"),
               len(new_offs) - 1)
        self._scratch[key] = hit
        return hit

    def scratch(self, name, n, dtype):
        torch = _torch()
        t = self._scratch.get(name)
        if t is None or t.numel() < n or t.dtype != dtype:
            t = torch.zeros(max(n, 1), dtype=dtype, device="cuda")
            self._scratch[name] = t
        return t

    def static_speed(self):
        """Per patch (x, y): the largest material speed of the cells the CFL
        face ranges touch (solver.py:457-460).  Equal to the per-face |speed|
        maximum whenever no cell is dry; cached on the device."""
        if getattr(self, "_static_speed", None) is None:
            g = self.g
            sp = np.zeros((len(self.patches), 2))
            for k, p in enumerate(self.patches):
                c = np.asarray(p.aux.c, dtype=float)
                if self.ndim == 2:
                    sp[k, 0] = np.max(c[g - 1:c.shape[0] - g + 1, g:c.shape[1] - g])
                    sp[k, 1] = np.max(c[g:c.shape[0] - g, g - 1:c.shape[1] - g + 1])
                else:
                    sp[k, 0] = np.max(c[g - 1:c.shape[0] - g + 1])
            self._static_speed_np = sp
            self._static_speed = _torch().from_numpy(sp.reshape(-1).copy()).to("cuda")
        return self._static_speed

    def static_speed_np(self):
        self.static_speed()
        return self._static_speed_np

    def job_classes(self, tiles, ntile, jobs, njob):
        """Per warp job of a FAST job table (ADJ_STEP_WET_DRY): 0 when every
        cell its strips read is wet (the all-wet march), 2 when every output
        cell is dry (copied), 1 otherwise; cached per table (materials are
        static)."""
        key = ("job_class", _ptr(tiles), ntile, _ptr(jobs) if jobs is not None else 0, njob)
        hit = self._scratch.get(key)
        if hit is not None:
            return hit
        rows = np.frombuffer(tiles.cpu().numpy().tobytes(), dtype=_lib.TILE_DTYPE)[:ntile]
        offs = (jobs.cpu().numpy().astype(np.int64) if jobs is not None
                else np.arange(ntile + 1, dtype=np.int64))
        wet = [np.asarray(p.aux.c) > 0.0 for p in self.patches]
        g = self.g
        tcls = np.empty(ntile, dtype=np.int8)
        for t, r in enumerate(rows):
            w = wet[int(r["patch"])]
            i0, j0, ni, nj = int(r["i0"]), int(r["j0"]), int(r["ni"]), int(r["nj"])
            if w[i0:i0 + ni + 2 * g, j0:j0 + nj + 2 * g].all():
                tcls[t] = 0
            elif not w[i0 + g:i0 + g + ni, j0 + g:j0 + g + nj].any():
                tcls[t] = 2
            else:
                tcls[t] = 1
        jcls = np.ones(len(offs) - 1, dtype=np.int8)
        for j in range(len(offs) - 1):
            c = tcls[offs[j]:offs[j + 1]]
            jcls[j] = 0 if (c == 0).all() else (2 if (c == 2).all() else 1)
        dev = _torch().from_numpy(jcls).to("cuda")
        self._scratch[key] = dev
        return dev

    # per-job materials are classified on the host, one window reduction per strip: levels of
    # many patches (AMR regrids rebuild their tables often) keep the per-cell march
    JOB_UNIFORM_MAX_PATCHES = 16
    JOB_UNIFORM_MIN_SHARE = 0.25

    def job_uniform(self, tiles, ntile, jobs, njob):
        """Per warp job of a FAST job table (ADJ_STEP_UNIFORM_MAT, acoustics):
        the (c, z) of every cell the job's strips read when they all hold one
        material, else (0, 0); None when too few jobs qualify (or the level has
        too many patches to classify on the host).  Cached per table."""
        if not USE_UNIFORM_MAT or self.swe or self.ndim != 2 or len(self.patches) > self.JOB_UNIFORM_MAX_PATCHES:
            return None
        key = ("job_uniform", _ptr(tiles), ntile, _ptr(jobs) if jobs is not None else 0, njob)
        if key in self._scratch:
            return self._scratch[key]
        if _torch().cuda.is_current_stream_capturing():
            return None           # the classification downloads the job table: not during a capture
        rows = np.frombuffer(tiles.cpu().numpy().tobytes(), dtype=_lib.TILE_DTYPE)[:ntile]
        offs = (jobs.cpu().numpy().astype(np.int64) if jobs is not None
                else np.arange(ntile + 1, dtype=np.int64))
        cz = [(np.asarray(p.aux.planes()[0]), np.asarray(p.aux.planes()[1])) for p in self.patches]
        g = self.g
        tu = np.zeros((ntile, 2))
        for t, r in enumerate(rows):
            c, z = cz[int(r["patch"])]
            i0, j0, ni, nj = int(r["i0"]), int(r["j0"]), int(r["ni"]), int(r["nj"])
            cw, zw = c[i0:i0 + ni + 2 * g, j0:j0 + nj + 2 * g], z[i0:i0 + ni + 2 * g, j0:j0 + nj + 2 * g]
            c0, z0 = float(cw.flat[0]), float(zw.flat[0])
            if c0 > 0.0 and z0 > 0.0 and cw.min() == c0 and cw.max() == c0 and zw.min() == z0 and zw.max() == z0:
                tu[t] = (c0, z0)
        ju = np.zeros((len(offs) - 1, 2))
        for j in range(len(offs) - 1):
            u = tu[offs[j]:offs[j + 1]]
            if u[0, 0] > 0.0 and np.all(u == u[0]):
                ju[j] = u[0]
        dev = None
        if np.count_nonzero(ju[:, 0]) >= self.JOB_UNIFORM_MIN_SHARE * len(ju):
            dev = _torch().from_numpy(np.ascontiguousarray(ju.reshape(-1))).to("cuda")
            self._scratch[("job_uniform_np", _ptr(tiles))] = ju
        self._scratch[key] = dev
        return dev

    def any_dry(self) -> bool:
        """Whether any cell of the level is dry (cached; materials are static
        and re-sampled only through sample_patch_material, which resets it)."""
        if not self.swe:
            return False
        if self._dry is None:
            self._dry = any(bool(np.any(~p.aux.wet)) for p in self.patches)
        return self._dry


def fast_dry_ok(store: LevelStore, equation) -> bool:
    """Whether the FAST strip kernel steps this level although it has dry
    cells: shallow water, forward (wave form) or the time-reversed f-wave
    adjoint, 2D, one row per lane (ADJ_STEP_WET_DRY)."""
    return (store.swe and store.ndim == 2 and not store.two_rows() and
            tuple(equation.kernel_spec()) in ((_lib.SYS_SWE2D, _lib.FORM_WAVE, 0), (_lib.SYS_SWE2D, _lib.FORM_FWAVE, 1)))


def fast_static(store: LevelStore, equation, variant) -> bool:
    """The FAST static-CFL path applies: 2D, and no dry cell or the wet/dry
    strip kernel (the static per-patch bound equals the reference's face
    maximum there too: a wet/dry face moves at the wet side's speed, a
    both-dry face not at all, and dry cells have c = 0)."""
    return (variant == _lib.VARIANT_FAST and store.ndim == 2 and
            (not store.any_dry() or fast_dry_ok(store, equation)))


# ---------------------------------------------------------------------------
# launch wrappers


def ring_copy(store: LevelStore, src, dst, stream=None):
    """Copy every patch's ghost ring from buffer src to buffer dst."""
    if SHADOW:
        return
    tab = store._scratch.get("ring_rects")      # the store's patch set is fixed: build the table once
    if tab is None:
        rects = []
        g = store.g
        for k, (off, NX, NY, pitch) in enumerate(store.boxes):
            if store.ndim == 2:
                parts = [(0, 0, g, NY), (NX - g, 0, g, NY), (g, 0, NX - 2 * g, g), (g, NY - g, NX - 2 * g, g)]
            else:
                parts = [(0, 0, g, 1), (NX - g, 0, g, 1)]
            for (i0, j0, ni, nj) in parts:
                rects.append((_lib.RECT_COPY, k, k, i0, j0, ni, nj, i0, j0, 0))
        tab = store._scratch["ring_rects"] = RectTable(np.array(rects, dtype=_lib.RECT_DTYPE))
    copy_rects(store, store, tab, src, dst, stream)


class RectTable:
    """A rectangle list resident on the device (built once per regrid).
    With ``coarse_geom`` = (fine_store, coarse_store, hierarchy) the
    interpolation weights of every COARSE rect are precomputed per row and
    column (``axis_weights``) and stored alongside."""

    MAX_CELLS = 256     # one warp per rectangle: large rectangles are split

    def __init__(self, rects_np, coarse_geom=None):
        rects_np = self._split(np.array(rects_np, dtype=_lib.RECT_DTYPE))
        self.n = len(rects_np)
        self.max_cells = int(np.max(rects_np["ni"] * rects_np["nj"])) if self.n else 0
        self.axis_w = self.axis_i = None
        if coarse_geom is not None and self.n:
            w, i = axis_weight_tables(rects_np, *coarse_geom)
            torch = _torch()
            self.axis_w = torch.from_numpy(w).to("cuda")
            self.axis_i = torch.from_numpy(i).to("cuda")
        self.dev = _dev_table(rects_np) if self.n else None
        self.np = rects_np

    @classmethod
    def _split(cls, rects):
        """Split rectangles larger than MAX_CELLS into row / column chunks
        (same cells, so the result is unchanged).  Vectorised: rect r becomes
        ceil(ni/ci) x ceil(nj/cj) chunks in row-major chunk order."""
        if len(rects) == 0 or int(np.max(rects["ni"] * rects["nj"])) <= cls.MAX_CELLS:
            return rects
        ni = rects["ni"].astype(np.int64)
        nj = rects["nj"].astype(np.int64)
        cj = np.minimum(nj, cls.MAX_CELLS)
        ci = np.maximum(1, cls.MAX_CELLS // cj)
        na = -(-ni // ci)
        nb = -(-nj // cj)
        cnt = na * nb
        src = np.repeat(np.arange(len(rects)), cnt)
        k = np.arange(int(cnt.sum())) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        a = (k // nb[src]) * ci[src]
        b = (k % nb[src]) * cj[src]
        out = rects[src].copy()
        out["di0"] += a.astype(np.int32)
        out["dj0"] += b.astype(np.int32)
        out["si0"] += a.astype(np.int32)
        out["sj0"] += b.astype(np.int32)
        out["ni"] = np.minimum(ci[src], ni[src] - a)
        out["nj"] = np.minimum(cj[src], nj[src] - b)
        return out


def _axis_weights_np(coord, origin, width, n):
    """_axis_weights (geometry.py:248-260), vectorised, same IEEE operations."""
    s = (coord - origin) / width - 0.5
    i0 = np.floor(s).astype(np.int64)
    w = s - i0
    w = np.where(i0 < 0, 0.0, np.where(i0 > n - 2, 1.0, w))
    i0 = np.clip(i0, 0, max(n - 2, 0))
    if n == 1:
        w = np.zeros_like(w)
    return i0, w


def axis_weight_tables(rects, fine_store, coarse_store, hierarchy):
    """Per COARSE rect: x weights of its rows then y weights of its columns;
    sets rects["pad"] to the rect's offset into the tables.  Vectorised over
    all rects; every element sees the same IEEE operations as
    ``_axis_weights_np`` (geometry.py:248-260)."""
    level = fine_store.patches[0].spec.level
    wf = hierarchy.widths(level)
    wc = hierarchy.widths(level - 1)
    org = hierarchy.origin
    gf, gc = fine_store.g, coarse_store.g
    sel = np.nonzero(rects["kind"] == _lib.RECT_COARSE)[0]
    if len(sel) == 0:
        return np.zeros(1), np.zeros(1, np.int32)
    nd = fine_store.ndim
    dlo = np.array([p.spec.lo for p in fine_store.patches], dtype=np.int64).reshape(-1, nd)
    slo = np.array([p.spec.lo for p in coarse_store.patches], dtype=np.int64).reshape(-1, nd)
    sshape = np.array([p.spec.shape for p in coarse_store.patches], dtype=np.int64).reshape(-1, nd)
    r = rects[sel]
    dpi = r["dst_patch"].astype(np.int64)
    spi = r["src_patch"].astype(np.int64)
    lens = [r["ni"].astype(np.int64)] + ([r["nj"].astype(np.int64)] if nd == 2 else [])
    d0s = [r["di0"].astype(np.int64)] + ([r["dj0"].astype(np.int64)] if nd == 2 else [])
    per_rect = lens[0] + (lens[1] if nd == 2 else 0)
    offs = np.cumsum(per_rect) - per_rect
    rects["pad"][sel] = offs.astype(rects["pad"].dtype)
    total = int(per_rect.sum())
    W = np.empty(total, np.float64)
    I = np.empty(total, np.int32)
    for ax in range(nd):
        n = lens[ax]
        base = offs + (lens[0] if ax == 1 else 0)
        rid = np.repeat(np.arange(len(sel)), n)
        t = np.arange(int(n.sum())) - np.repeat(np.cumsum(n) - n, n)
        gidx = dlo[dpi[rid], ax] - gf + d0s[ax][rid] + t
        coord = org[ax] + (gidx + 0.5) * wf[ax]
        lo_phys = org[ax] + (slo[spi[rid], ax] - gc) * wc[ax]
        ncell = sshape[spi[rid], ax] + 2 * gc
        s = (coord - lo_phys) / wc[ax] - 0.5
        i0 = np.floor(s).astype(np.int64)
        w = s - i0
        w = np.where(i0 < 0, 0.0, np.where(i0 > ncell - 2, 1.0, w))
        i0 = np.clip(i0, 0, np.maximum(ncell - 2, 0))
        w = np.where(ncell == 1, 0.0, w)
        pos = base[rid] + t
        W[pos] = w
        I[pos] = i0.astype(np.int32)
    return W, I


def _as_table(rects):
    return rects if isinstance(rects, RectTable) else RectTable(rects)


def copy_rects(dst_store, src_store, rects_np, src_buf, dst_buf, stream=None):
    tab = _as_table(rects_np)
    if tab.n == 0 or SHADOW:
        return
    rects = tab.dev
    a = _lib.AdjGhostArgs()
    a.q_dst = _ptr(dst_buf)
    a.q_src = _ptr(src_buf)
    a.dst_patches = _ptr(dst_store.table)
    a.src_patches = _ptr(src_store.table)
    a.rects = _ptr(rects)
    a.dst_comp_stride = dst_store.plane
    a.src_comp_stride = src_store.plane
    a.nrect = tab.n
    a.ndim = dst_store.ndim
    a.m = dst_store.m
    a.ghost_dst = dst_store.g
    a.ghost_src = src_store.g
    a.ratio = 1
    a.time_mode = 0
    a.max_rect_cells = tab.max_cells
    a.stream = _lib.stream_ptr(stream)
    _lib.check(_lib.lib().adj_fill_ghost_rects(_lib.C.byref(a)), "adj_fill_ghost_rects")


def coarse_rects(fine_store, coarse_store, rects_np, q_old, q_new, hierarchy, ratio, w_time, mode,
                 dst_buf=None, stream=None, copy_src=None, copy_patches=None):
    """COARSE rects (and, when given, disjoint same-level COPY rects in the
    same launch, sourced from ``copy_src`` with the fine store's layout)."""
    tab = _as_table(rects_np)
    if tab.n == 0:
        return
    wptr = 0
    if PARAMS is not None:          # captured sweep: the weight (mode) is read from device memory
        if mode == 2:
            raise RuntimeError("coarse patches without saved state cannot be graph-replayed")
        wptr = PARAMS.take(w_time if mode == 1 else -1.0)
    if SHADOW:
        return
    rects = tab.dev
    fine_level = fine_store.patches[0].spec.level
    wf = hierarchy.widths(fine_level)
    wc = hierarchy.widths(fine_level - 1)
    org = hierarchy.origin
    a = _lib.AdjGhostArgs()
    a.q_dst = _ptr(dst_buf if dst_buf is not None else fine_store.buf[fine_store.cur])
    a.q_src = _ptr(copy_src)
    a.q_coarse_old = _ptr(q_old)
    a.q_coarse_new = _ptr(q_new)
    a.dst_patches = _ptr(fine_store.table)
    a.src_patches = _ptr(copy_patches)
    a.coarse_patches = _ptr(coarse_store.table)
    a.rects = _ptr(rects)
    a.dst_comp_stride = fine_store.plane
    a.src_comp_stride = fine_store.plane
    a.coarse_comp_stride = coarse_store.plane
    a.nrect = tab.n
    a.ndim = fine_store.ndim
    a.m = fine_store.m
    a.ghost_dst = fine_store.g
    a.ghost_src = coarse_store.g
    a.ratio = ratio
    a.origin_x = org[0]
    a.origin_y = org[1] if fine_store.ndim == 2 else 0.0
    a.dx_f, a.dy_f = wf[0], wf[1]
    a.dx_c, a.dy_c = wc[0], wc[1]
    a.w_time = w_time
    a.w_time_dev = wptr
    a.axis_w = _ptr(tab.axis_w)
    a.axis_i = _ptr(tab.axis_i)
    a.time_mode = mode
    a.max_rect_cells = tab.max_cells
    a.stream = _lib.stream_ptr(stream)
    _lib.check(_lib.lib().adj_fill_ghost_rects(_lib.C.byref(a)), "adj_fill_ghost_rects")


def _bc_codes(boundary):
    return tuple(_lib.BC_CODES[sd] for sd in (boundary.left, boundary.right, boundary.bottom, boundary.top))


def check_periodic(store, boundary, level_shape):
    """Periodic sides (an extension; the reference has wall and outflow) wrap
    a patch's ghosts to its own opposite interior, so every patch of the
    level must span each periodic axis."""
    for axis in range(store.ndim):
        if boundary.side(axis, False) != "periodic":
            continue
        for p in store.patches:
            if p.spec.lo[axis] != 0 or p.spec.hi[axis] != level_shape[axis] - 1:
                raise ValueError("periodic boundaries need every patch to span the periodic axis")


def physical_cell_count(store: LevelStore, level_shape) -> int:
    """Out-of-domain ghost cells of every patch (what the physical phase writes)."""
    g = store.g
    tot = 0
    for p in store.patches:
        s = p.spec
        full = 1
        ind = 1
        for ax in range(store.ndim):
            full *= s.shape[ax] + 2 * g
            ind *= min(s.hi[ax] + g, level_shape[ax] - 1) - max(s.lo[ax] - g, 0) + 1
        tot += full - ind
    return int(tot)


class GhostPlan:
    """Whole-level ghost fill as one gather launch (adj_ghost_plan_build /
    adj_fill_ghost_plan): the level's disjoint COARSE + COPY rectangles and
    its physical boundary cells, compiled on the device once per regrid.
    Same values as the coarse -> copy -> physical phases
    (fill_level_ghosts, amr.py:479-491)."""

    def __init__(self, store: LevelStore, rects: RectTable, coarse_store, boundary, equation, level_shape):
        torch = _torch()
        if "periodic" in (boundary.left, boundary.right, boundary.bottom, boundary.top):
            check_periodic(store, boundary, level_shape)
        r = rects.np if rects.n else np.zeros(0, dtype=_lib.RECT_DTYPE)
        kinds = r["kind"]
        is_c = kinds == _lib.RECT_COARSE
        if len(r) > 1 and np.any(is_c[1:] & ~is_c[:-1]):
            raise ValueError("GhostPlan needs COARSE rects before COPY rects")
        cells = (r["ni"].astype(np.int64) * r["nj"].astype(np.int64))
        cell0 = np.zeros(len(r) + 1, dtype=np.int64)
        np.cumsum(cells, out=cell0[1:])
        rect_cells = int(cell0[-1])
        nc = int(cells[kinds == _lib.RECT_COARSE].sum())
        store.edges_table(level_shape)
        edge_tab, nedge = store._edge_tab
        nphys = physical_cell_count(store, level_shape) if nedge else 0
        n = rect_cells + nphys
        self.n, self.nc = n, nc
        i32, f64 = torch.int32, torch.float64
        self.dst = torch.empty(max(n, 1), dtype=i32, device="cuda")
        self.src = torch.empty(max(n, 1), dtype=i32, device="cuda")
        self.meta = torch.empty(max(n, 1), dtype=i32, device="cuda")
        self.c_base = torch.empty(max(nc, 1), dtype=i32, device="cuda")
        self.c_step = torch.empty(max(nc, 1), dtype=i32, device="cuda")
        self.c_wx = torch.empty(max(nc, 1), dtype=f64, device="cuda")
        self.c_wy = torch.empty(max(nc, 1), dtype=f64, device="cuda")
        self.plan = _lib.AdjGhostPlan()
        for k in ("dst", "src", "meta", "c_base", "c_step", "c_wx", "c_wy"):
            setattr(self.plan, k, _ptr(getattr(self, k)))
        self.plan.n, self.plan.nc = n, nc
        if n == 0:
            return
        counter = torch.zeros(1, dtype=i32, device="cuda")
        owner = torch.full((store.plane,), -1, dtype=i32, device="cuda") if nphys else None
        cell0_dev = torch.from_numpy(cell0.astype(np.int32)).to("cuda")
        a = _lib.AdjGhostPlanBuildArgs()
        a.plan = self.plan
        a.rects = _ptr(rects.dev) if rects.n else 0
        a.rect_cell0 = _ptr(cell0_dev)
        a.patches = _ptr(store.table)
        a.coarse_patches = _ptr(coarse_store.table) if coarse_store is not None else 0
        a.axis_w = _ptr(rects.axis_w)
        a.axis_i = _ptr(rects.axis_i)
        a.edge_patches = _ptr(edge_tab) if nedge else 0
        a.owner = _ptr(owner)
        a.counter = _ptr(counter)
        a.nrect = rects.n
        a.rect_cells = rect_cells
        a.nedge = nedge
        a.ndim = store.ndim
        a.m = store.m
        a.ghost = store.g
        a.ghost_coarse = coarse_store.g if coarse_store is not None else 0
        a.max_ghost_cells = store.max_ghost_cells
        for k, code in enumerate(_bc_codes(boundary)):
            a.bc[k] = code
        a.normal_comp[0] = equation.normal_component(0)
        a.normal_comp[1] = equation.normal_component(1) if store.ndim == 2 else -1
        a.stream = _lib.stream_ptr(None)
        _lib.check(_lib.lib().adj_ghost_plan_build(_lib.C.byref(a)), "adj_ghost_plan_build")
        got = int(counter.item())
        if got != nphys:
            raise RuntimeError(f"ghost plan: {got} physical cells, expected {nphys}")

    @staticmethod
    def usable(store: LevelStore, coarse_store) -> bool:
        """Entries are 32-bit plane offsets."""
        lim = 2 ** 31 - 1
        return store.plane < lim and (coarse_store is None or coarse_store.plane < lim)

    def fill_args(self, store: LevelStore, q_old=None, q_new=None, coarse_store=None, w_time=0.0, mode=0,
                  stream=None):
        """The fill as an argument struct (for a standalone launch or a step
        prefill); takes the captured-sweep weight slot like fill()."""
        wptr = 0
        if PARAMS is not None and self.nc:      # captured sweep: weight read from device memory
            if mode == 2:
                raise RuntimeError("coarse patches without saved state cannot be graph-replayed")
            wptr = PARAMS.take(w_time if mode == 1 else -1.0)
        a = _lib.AdjGhostPlanFillArgs()
        a.plan = self.plan
        a.q = _ptr(store.buf[store.cur])
        a.q_coarse_old = _ptr(q_old)
        a.q_coarse_new = _ptr(q_new)
        a.comp_stride = store.plane
        a.coarse_comp_stride = coarse_store.plane if coarse_store is not None else 0
        a.ndim = store.ndim
        a.m = store.m
        a.time_mode = mode
        a.w_time = w_time
        a.w_time_dev = wptr
        a.stream = _lib.stream_ptr(stream)
        return a

    def fill(self, store: LevelStore, q_old=None, q_new=None, coarse_store=None, w_time=0.0, mode=0, stream=None):
        wptr = 0
        if PARAMS is not None and self.nc:      # captured sweep: weight read from device memory
            if mode == 2:
                raise RuntimeError("coarse patches without saved state cannot be graph-replayed")
            wptr = PARAMS.take(w_time if mode == 1 else -1.0)
        if SHADOW or self.n == 0:
            return
        a = _lib.AdjGhostPlanFillArgs()
        a.plan = self.plan
        a.q = _ptr(store.buf[store.cur])
        a.q_coarse_old = _ptr(q_old)
        a.q_coarse_new = _ptr(q_new)
        a.comp_stride = store.plane
        a.coarse_comp_stride = coarse_store.plane if coarse_store is not None else 0
        a.ndim = store.ndim
        a.m = store.m
        a.time_mode = mode
        a.w_time = w_time
        a.w_time_dev = wptr
        a.stream = _lib.stream_ptr(stream)
        _lib.check(_lib.lib().adj_fill_ghost_plan(_lib.C.byref(a)), "adj_fill_ghost_plan")


class JobFill:
    """A level's planned ghost fill (GhostPlan) regrouped by the FAST step's
    warp jobs (AdjJobFill): every job gets the plan entries whose ghost cell
    lies in the window its strips read (rows j0-2 .. j0+nj+1, columns
    i0-2 .. i0+ni+1 of the tile, ghost-inclusive), COARSE entries with their
    stencil inline.  The step launch then fills and marches in one kernel
    (no separate gather launch).  Built once per plan, on the host, from the
    device plan; only for levels of small patches (at most MAX_TILES strip
    tiles per patch)."""

    MAX_TILES = 16

    @staticmethod
    def usable(store: LevelStore) -> bool:
        if store.ndim != 2 or store.two_rows():
            return False
        tiles, ntile, jobs, njob = store.tiles(_lib.VARIANT_FAST)
        if jobs is None or ntile == 0:
            return False
        rows = store.__dict__.get("_tile_rows")
        if rows is None:
            rows = np.frombuffer(tiles.cpu().numpy().tobytes(), dtype=_lib.TILE_DTYPE)[:ntile].copy()
            store._tile_rows = rows
        return int(np.bincount(rows["patch"], minlength=len(store.patches)).max()) <= JobFill.MAX_TILES

    def __init__(self, store: LevelStore, gp: "GhostPlan"):
        torch = _torch()
        tiles, ntile, jobs, njob = store.tiles(_lib.VARIANT_FAST)
        rows = store._tile_rows
        offs_job = jobs.cpu().numpy().astype(np.int64)
        n, nc = gp.n, gp.nc
        dst = gp.dst[:n].cpu().numpy().astype(np.int64)
        src = gp.src[:n].cpu().numpy()
        meta = gp.meta[:n].cpu().numpy().view(np.uint32)
        isc = (meta & 1) != 0
        # owning patch and ghost-inclusive local cell of every entry
        toff = store.table_np["offset"].astype(np.int64)
        tpitch = store.table_np["pitch"].astype(np.int64)
        k = np.searchsorted(toff, dst, side="right") - 1
        rem = dst - toff[k]
        ii, jj = rem // tpitch[k], rem % tpitch[k]
        # candidate tiles of the entry's patch
        order = np.argsort(rows["patch"], kind="stable")
        cnt = np.bincount(rows["patch"], minlength=len(store.patches))
        first = np.zeros(len(cnt) + 1, dtype=np.int64)
        np.cumsum(cnt, out=first[1:])
        g = store.g
        ent, tix = [], []
        for t in range(int(cnt.max()) if len(cnt) else 0):
            sel = np.flatnonzero(cnt[k] > t)
            tt = order[first[k[sel]] + t]
            r = rows[tt]
            i0, j0 = g + r["i0"].astype(np.int64), g + r["j0"].astype(np.int64)
            inside = ((ii[sel] >= i0 - 2) & (ii[sel] < i0 + r["ni"] + 2) &
                      (jj[sel] >= j0 - 2) & (jj[sel] < j0 + r["nj"] + 2))
            ent.append(sel[inside])
            tix.append(tt[inside])
        ent = np.concatenate(ent) if ent else np.zeros(0, np.int64)
        tix = np.concatenate(tix) if tix else np.zeros(0, np.int64)
        job = np.searchsorted(offs_job, tix, side="right") - 1
        o = np.lexsort((ent, job))
        ent, job = ent[o], job[o]
        self.n = m = len(ent)
        self.nc = int(isc[ent].sum()) if m else 0
        entry_off = np.searchsorted(job, np.arange(njob + 1)).astype(np.int32)
        i32, f64 = torch.int32, torch.float64
        up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
        self.entry_off = up(entry_off, i32)
        self.dst = up(dst[ent].astype(np.int32), i32)
        self.src = up(src[ent].astype(np.int32), i32)
        self.meta = up(meta[ent].view(np.int32), i32)
        self.c_base = self.c_step = self.c_wx = self.c_wy = self.cache = None
        if nc and self.nc:
            # own coarse stencil (rect COARSE entries e < nc) or the mirrored entry's (physical)
            e = ent
            ci = np.where(e < nc, e, src[e])
            ci = np.where(isc[e], ci, 0)
            self.c_base = up(gp.c_base[:nc].cpu().numpy()[ci], i32)
            self.c_step = up(gp.c_step[:nc].cpu().numpy()[ci], i32)
            self.c_wx = up(gp.c_wx[:nc].cpu().numpy()[ci], f64)
            self.c_wy = up(gp.c_wy[:nc].cpu().numpy()[ci], f64)
            self.cache = torch.zeros(6 * max(m, 1), dtype=f64, device="cuda")
        self.cache_key = None     # the coarse interval whose values the cache holds

    def args(self, q_old=None, q_new=None, coarse_store=None, w_time=0.0, mode=0, cache_mode=0):
        """The AdjJobFill struct of one step launch (takes the captured-sweep
        weight slot like GhostPlan.fill_args)."""
        wptr = 0
        if PARAMS is not None and self.c_base is not None:
            if mode == 2:
                raise RuntimeError("coarse patches without saved state cannot be graph-replayed")
            wptr = PARAMS.take(w_time if mode == 1 else -1.0)
        f = _lib.AdjJobFill()
        f.entry_off, f.dst, f.src, f.meta = (_ptr(self.entry_off), _ptr(self.dst), _ptr(self.src), _ptr(self.meta))
        if self.c_base is not None:
            f.c_base, f.c_step, f.c_wx, f.c_wy = (_ptr(self.c_base), _ptr(self.c_step), _ptr(self.c_wx),
                                                  _ptr(self.c_wy))
            f.cache = _ptr(self.cache)
            f.cache_mode = cache_mode
            f.q_coarse_old, f.q_coarse_new = _ptr(q_old), _ptr(q_new)
            f.coarse_comp_stride = coarse_store.plane
        f.n = self.n
        f.time_mode = mode
        f.w_time = w_time
        f.w_time_dev = wptr
        return f


def fill_physical(store: LevelStore, boundary, equation, level_shape, stream=None, slots=None):
    """K2 physical phase on every patch of the store (solver.py:125-146);
    ``slots`` restricts it to a subset of patches."""
    store.sync_in(stream)
    store.edges_table(level_shape)
    table, nedge = store._edge_tab
    if nedge == 0:
        return
    full = store.all_edges_physical(level_shape)
    if slots is not None:
        sub = store.table_np.copy()
        keep = np.zeros(len(sub), dtype=bool)
        keep[list(slots)] = True
        sub["edges"][~keep] = 0
        sub = sub[sub["edges"] != 0]
        table, nedge = _dev_table(sub), len(sub)
        full = full and bool(np.all(keep))
        if nedge == 0:
            return
    if "periodic" in (boundary.left, boundary.right, boundary.bottom, boundary.top):
        check_periodic(store, boundary, level_shape)
    store.prepare_write(full_ghosts=full, stream=stream)
    if SHADOW:
        return
    a = _lib.AdjPhysArgs()
    a.q = _ptr(store.buf[store.cur])
    a.patches = _ptr(table)
    a.comp_stride = store.plane
    a.npatch = nedge
    a.ndim = store.ndim
    a.ghost = store.g
    a.m = store.m
    sides = (boundary.left, boundary.right, boundary.bottom, boundary.top)
    for k, sd in enumerate(sides):
        a.bc[k] = _lib.BC_CODES[sd]
    a.normal_comp[0] = equation.normal_component(0)
    a.normal_comp[1] = equation.normal_component(1) if store.ndim == 2 else -1
    a.max_ghost_cells = store.max_ghost_cells
    a.stream = _lib.stream_ptr(stream)
    _lib.check(_lib.lib().adj_fill_physical(_lib.C.byref(a)), "adj_fill_physical")


def launch_step(store: LevelStore, dt, equation, limiter, variant, out_buf_index, stream=None,
                accumulate=False, prefill=None, fine_restrict=None, job_fill=None, phys_in=None):
    """K1 on every patch: reads buf[cur], writes buf[out_buf_index].
    Returns (speed_max (npatch, 2) tensor, nonfinite (npatch,) tensor).
    ``accumulate`` (static-CFL fast path only): no per-launch memsets; the
    non-finite flags accumulate in ``store.nonfinite_acc`` and speed_max is
    not written (the caller uses the static bound)."""
    if limiter not in _lib.LIMITERS:
        raise ValueError(f"unknown limiter {limiter!r}")
    torch = _torch()
    npatch = len(store.patches)
    wet_dry = False
    if variant == _lib.VARIANT_FAST and store.any_dry():
        # dry cells: the strip kernel's wet/dry instantiation (forward shallow water, no fused
        # restriction or in-launch fill); anything else steps with the EXACT kernel
        if fast_dry_ok(store, equation) and fine_restrict is None and prefill is None and job_fill is None:
            wet_dry = True
        else:
            variant = _lib.VARIANT_EXACT
    tiles, ntile, jobs, njob = store.tiles(variant)
    if phys_in is not None:          # jobs that fill physical ghosts go first
        tiles, ntile, jobs, njob = store.tiles_edge_first(phys_in[2])
    smax = store.scratch("smax", 2 * npatch, torch.float64)
    accumulate = accumulate and variant == _lib.VARIANT_FAST and store.ndim == 2
    if accumulate:
        if store.nonfinite_acc is None:
            store.nonfinite_acc = torch.zeros(npatch, dtype=torch.int32, device="cuda")
        bad = store.nonfinite_acc
    else:
        bad = store.scratch("nonfinite", npatch, torch.int32)
    counter = store.scratch("work_counter", 4, torch.int32)   # zero; kept zero by the FAST kernel
    if SHADOW:
        return smax[: 2 * npatch].view(npatch, 2), bad[:npatch]
    system, form, rev = equation.kernel_spec()
    spec0 = store.patches[0].spec
    a = _lib.AdjStepArgs()
    a.q_in = _ptr(store.buf[store.cur])
    a.q_out = _ptr(store.buf[out_buf_index])
    a.aux = _ptr(store.aux)
    a.patches = _ptr(store.table)
    a.tiles = _ptr(tiles)
    a.speed_max = _ptr(smax)
    a.nonfinite = _ptr(bad)
    a.work_counter = _ptr(counter)
    a.static_speed = _ptr(store.static_speed()) if variant == _lib.VARIANT_FAST and store.ndim == 2 else 0
    a.job_offsets = _ptr(jobs)
    a.njob = njob
    a.comp_stride = store.plane
    a.aux_stride = store.plane
    a.npatch = npatch
    a.ntile = ntile
    a.ndim = store.ndim
    a.ghost = store.g
    a.system, a.form, a.reversed = system, form, rev
    a.limiter = _lib.LIMITERS[limiter]
    a.variant = variant
    a.flags = (_lib.STEP_KEEP_NONFINITE | _lib.STEP_NO_SPEED_OUT) if accumulate else 0
    if variant == _lib.VARIANT_FAST and store.ndim == 2:
        a.flags |= _lib.STEP_COUNTER_ZERO
        if store.two_rows():
            a.flags |= _lib.STEP_TWO_ROWS
        if store.uniform_mat is not None and a.static_speed:
            a.flags |= _lib.STEP_UNIFORM_MAT
            a.uniform_c, a.uniform_z = store.uniform_mat
        elif a.static_speed and not wet_dry and (system, form, rev) == (_lib.SYS_AC2D, _lib.FORM_WAVE, 0):
            ju = store.job_uniform(tiles, ntile, jobs, njob)
            if ju is not None:
                a.flags |= _lib.STEP_UNIFORM_MAT
                a.job_uniform = _ptr(ju)
        if wet_dry:
            a.flags |= _lib.STEP_WET_DRY
            if USE_JOB_CLASS:
                a.job_class = _ptr(store.job_classes(tiles, ntile, jobs, njob))
    a.dt = dt
    a.dtdx = dt / spec0.dx
    a.dtdy = dt / spec0.dy if store.ndim == 2 else 0.0
    a.gravity = equation.gravity
    a.stream = _lib.stream_ptr(stream)
    if prefill is not None:
        a.prefill = prefill
    if job_fill is not None:          # AdjJobFill: the level's ghost fill per warp job
        a.job_fill = job_fill
    if phys_in is not None:           # (boundary, equation, level shape): fill_ghost_physical of q_in inside the launch
        bd, eq = phys_in[0], phys_in[1]
        a.flags |= _lib.STEP_PHYS_IN
        for k, sd in enumerate((bd.left, bd.right, bd.bottom, bd.top)):
            a.phys_bc[k] = _lib.BC_CODES[sd]
        a.phys_normal[0] = eq.normal_component(0)
        a.phys_normal[1] = eq.normal_component(1)
    if fine_restrict is not None:     # (FusedRestrict, coarse store): restriction fused into this step
        fr, cst = fine_restrict
        a.fine_restrict.q_coarse = _ptr(cst.buf[cst.cur])
        a.fine_restrict.cell = _ptr(fr.cell)
        a.fine_restrict.base = _ptr(fr.base)
        a.fine_restrict.coarse_comp_stride = cst.plane
        a.fine_restrict.ratio = fr.ratio
    _lib.check(_lib.lib().adj_step_level(_lib.C.byref(a)), "adj_step_level")
    return smax[: 2 * npatch].view(npatch, 2), bad[:npatch]


def restrict_cells(coarse_store, fine_store, rects, ratio):
    """Planned restriction: per covered coarse cell (row-major within each
    overlap rect) its coarse offset, the offset of its first fine child and
    meta = flat | fine pitch << 1, from the UNSPLIT overlap rects (numpy's
    flat reduction order depends on the overlap box, amr.py:440-450)."""
    nd = coarse_store.ndim
    gC, gF = coarse_store.g, fine_store.g
    gCy, gFy = (gC, gF) if nd == 2 else (0, 0)
    rj = ratio if nd == 2 else 1
    ni = rects["ni"].astype(np.int64)
    nj = rects["nj"].astype(np.int64)
    cnt = ni * nj
    rid = np.repeat(np.arange(len(rects)), cnt)
    k = np.arange(int(cnt.sum())) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    a = k // nj[rid]
    b = k % nj[rid]
    ct = coarse_store.table_np
    ft = fine_store.table_np
    cp = rects["dst_patch"].astype(np.int64)[rid]
    fp = rects["src_patch"].astype(np.int64)[rid]
    cdst = ct["offset"][cp] + (gC + rects["di0"].astype(np.int64)[rid] + a) * ct["pitch"][cp].astype(np.int64) + \
        (gCy + rects["dj0"].astype(np.int64)[rid] + b)
    fpitch = ft["pitch"][fp].astype(np.int64)
    fsrc = ft["offset"][fp] + (gF + rects["si0"].astype(np.int64)[rid] + a * ratio) * fpitch + \
        (gFy + rects["sj0"].astype(np.int64)[rid] + b * rj)
    flat = (nd == 2) & (nj[rid] == 1)
    meta = flat.astype(np.int64) | (fpitch << 1)
    return cdst.astype(np.int32), fsrc.astype(np.int32), meta.astype(np.int32)


class RestrictPlan:
    """Device copy of restrict_cells (built once per regrid)."""

    def __init__(self, coarse_store, fine_store, rects_np, ratio):
        torch = _torch()
        d, s_, m = restrict_cells(coarse_store, fine_store, rects_np, ratio)
        self.n = len(d)
        self.dst = torch.from_numpy(d if self.n else np.zeros(1, np.int32)).to("cuda")
        self.src = torch.from_numpy(s_ if self.n else np.zeros(1, np.int32)).to("cuda")
        self.meta = torch.from_numpy(m if self.n else np.zeros(1, np.int32)).to("cuda")

    @staticmethod
    def usable(coarse_store, fine_store) -> bool:
        lim = 2 ** 31 - 1
        return coarse_store.plane < lim and fine_store.plane < lim


class FusedRestrict:
    """Restriction fused into the fine level's step (AdjStepRestrict): per
    fine r x r block (patch-major, then x block, then y block) the offset of
    its covered coarse cell in the coarse plane, -1 where not covered.
    Built once per regrid from restrict_cells."""

    def __init__(self, coarse_store, fine_store, rects_np, ratio):
        torch = _torch()
        d, s_, _ = restrict_cells(coarse_store, fine_store, rects_np, ratio)
        t = fine_store.table_np
        g = fine_store.g
        nbx, nby = t["nx"].astype(np.int64) // ratio, t["ny"].astype(np.int64) // ratio
        base = np.concatenate([[0], np.cumsum(nbx * nby)[:-1]]).astype(np.int64)
        cell = np.full(max(int((nbx * nby).sum()), 1), -1, dtype=np.int32)
        if len(d):
            offs = t["offset"].astype(np.int64)
            order = np.argsort(offs, kind="stable")
            k = order[np.searchsorted(offs[order], s_.astype(np.int64), side="right") - 1]
            xr, yr = np.divmod(s_.astype(np.int64) - offs[k], t["pitch"][k].astype(np.int64))
            cell[base[k] + ((xr - g) // ratio) * nby[k] + (yr - g) // ratio] = d
        self.ratio = ratio
        self.cell = torch.from_numpy(cell).to("cuda")
        self.base = torch.from_numpy(base.astype(np.int32)).to("cuda")

    @staticmethod
    def usable(coarse_store, fine_store, ratio) -> bool:
        """FAST 2D fine level without dry cells whose strip tiles all align to the ratio."""
        if ratio not in (2, 4) or fine_store.ndim != 2 or fine_store.any_dry() or fine_store.two_rows():
            return False
        if coarse_store.any_dry():      # shallow water restricts into wet coarse cells only
            return False
        if not RestrictPlan.usable(coarse_store, fine_store):
            return False
        key = ("fused_restrict_ok", ratio)
        ok = fine_store._scratch.get(key)
        if ok is None:
            tiles, ntile, _, _ = fine_store.tiles(_lib.VARIANT_FAST)
            rows = np.frombuffer(tiles.cpu().numpy().tobytes(), dtype=_lib.TILE_DTYPE)[:ntile]
            t = fine_store.table_np
            ok = bool(np.all(rows["i0"] % ratio == 0) and np.all(rows["j0"] % ratio == 0)
                      and np.all(rows["ni"] % ratio == 0) and np.all(rows["nj"] % ratio == 0)
                      and np.all(t["nx"] % ratio == 0) and np.all(t["ny"] % ratio == 0))
            fine_store._scratch[key] = ok
        return ok


def restrict_rects(coarse_store, fine_store, rects_np, ratio, swe, stream=None):
    plan = rects_np if isinstance(rects_np, RestrictPlan) else None
    tab = None if plan is not None else _as_table(rects_np)
    if (plan.n if plan is not None else tab.n) == 0 or SHADOW:
        return
    a = _lib.AdjRestrictArgs()
    if plan is not None:
        a.cell_dst, a.cell_src, a.cell_meta = _ptr(plan.dst), _ptr(plan.src), _ptr(plan.meta)
        a.ncell = plan.n
    else:
        a.rects = _ptr(tab.dev)
        a.nrect = tab.n
        a.max_rect_cells = tab.max_cells
    a.q_coarse = _ptr(coarse_store.buf[coarse_store.cur])
    a.q_fine = _ptr(fine_store.buf[fine_store.cur])
    a.aux_coarse = _ptr(coarse_store.aux)
    a.aux_fine = _ptr(fine_store.aux)
    a.coarse_patches = _ptr(coarse_store.table)
    a.fine_patches = _ptr(fine_store.table)
    a.coarse_comp_stride = coarse_store.plane
    a.fine_comp_stride = fine_store.plane
    a.coarse_aux_stride = coarse_store.plane
    a.fine_aux_stride = fine_store.plane
    a.ndim = coarse_store.ndim
    a.m = coarse_store.m
    a.ratio = ratio
    a.swe = int(swe)
    a.ghost_coarse = coarse_store.g
    a.ghost_fine = fine_store.g
    a.stream = _lib.stream_ptr(stream)
    _lib.check(_lib.lib().adj_restrict(_lib.C.byref(a)), "adj_restrict")


def region_tables(store: LevelStore, regions, t):
    """Per-patch row / column bitmasks of the refinement regions that act at
    time t on flags of this level (RefinementRegion.cell_mask and the
    force / clear order of flag_cells, amr.py:137-154).  Returns None when no
    region acts, else (rows, cols, row_off, col_off, force_bits, clear_bits);
    raises ValueError beyond 8 regions."""
    new_level = store.patches[0].spec.level + 1
    force = clear = 0
    for k, r in enumerate(regions):
        if not r.contains_time(t):
            continue
        if new_level <= r.min_level:
            force |= 1 << k
        if new_level > r.max_level:
            clear |= 1 << k
    if not (force | clear):
        return None
    if len(regions) > 8:
        raise ValueError("device region tables hold at most 8 regions")
    rows, cols, roff, coff = [], [], [], []
    nr = nc = 0
    for p in store.patches:
        cs = p.spec.cell_centers()
        rb = np.zeros(len(cs[0]), dtype=np.uint8)
        cb = np.zeros(len(cs[1]) if store.ndim == 2 else 0, dtype=np.uint8)
        for k, r in enumerate(regions):
            rb |= (((cs[0] >= r.rect[0]) & (cs[0] <= r.rect[1])).astype(np.uint8) << k)
            if store.ndim == 2:
                cb |= (((cs[1] >= r.rect[2]) & (cs[1] <= r.rect[3])).astype(np.uint8) << k)
        roff.append(nr)
        coff.append(nc)
        rows.append(rb)
        cols.append(cb)
        nr += len(rb)
        nc += len(cb)
    cat = lambda xs: np.concatenate(xs) if xs and sum(len(x) for x in xs) else np.zeros(1, np.uint8)
    return cat(rows), cat(cols), np.array(roff, np.int32), np.array(coff, np.int32), force, clear


def flag_level_mask(store: LevelStore, bits, level_shape, buffer_cells, regions=(), t=0.0, stream=None):
    """K5 on K3's packed flags of every patch of ``store``: -> (clipped bool
    mask, allowed bool mask, raw flag count after region overrides), both
    masks over the level's index space (amr.py:570-581)."""
    torch = _torch()
    nx = int(level_shape[0])
    ny = int(level_shape[1]) if store.ndim == 2 else 1
    mask = torch.empty(nx * ny, dtype=torch.uint8, device="cuda")
    occ = torch.empty(nx * ny, dtype=torch.uint8, device="cuda")
    raw = torch.empty(1, dtype=torch.int64, device="cuda")
    tabs = region_tables(store, regions, t) if regions else None
    keep = []
    a = _lib.AdjFlagMaskArgs()
    a.flag_bits = _ptr(bits)
    a.patches = _ptr(store.table)
    if tabs is not None:
        rows, cols, roff, coff, force, clear = tabs
        keep = [torch.from_numpy(x).to("cuda") for x in (rows, cols, roff, coff)]
        a.region_rows, a.region_cols, a.region_row_off, a.region_col_off = (_ptr(x) for x in keep)
        a.force_regions, a.clear_regions = force, clear
    a.mask = _ptr(mask)
    a.occupancy = _ptr(occ)
    a.raw_count = _ptr(raw)
    a.npatch = len(store.patches)
    a.ndim = store.ndim
    a.level_nx, a.level_ny = nx, ny
    a.buffer = int(buffer_cells)
    a.max_cells = max(int(np.prod(p.spec.shape)) for p in store.patches)
    a.stream = _lib.stream_ptr(stream)
    _lib.check(_lib.lib().adj_flag_level_mask(_lib.C.byref(a)), "adj_flag_level_mask")
    m = mask.cpu().numpy().reshape((nx, ny) if store.ndim == 2 else (nx,))
    del keep
    return (m & 1).astype(bool), (m & 2).astype(bool), int(raw.item())


def flag_axis_tables(store: LevelStore, ring_shape, a_origin, a_dx, a_dy, level_origin, level_dx, level_dy):
    """Per patch row/column bilinear weights into the adjoint grid, computed
    once with interpolate_uniform's arithmetic (geometry.py:248-290) and its
    bounds check (raises OutOfRangeError), plus _adjoint_dry_at indices
    (adjoint.py:217-224).  Cached per store and adjoint geometry."""
    key = ("flagtab", tuple(ring_shape), tuple(a_origin), a_dx, a_dy, tuple(level_origin), level_dx, level_dy)
    hit = store._scratch.get(key)
    if hit is not None:
        return hit
    from .geometry import OutOfRangeError
    nd = store.ndim
    n_a = [ring_shape[0]] + ([ring_shape[1]] if nd == 2 else [])
    widths_a = [a_dx] + ([a_dy] if nd == 2 else [])
    widths_f = [level_dx] + ([level_dy] if nd == 2 else [])
    hi0 = a_origin[0] + n_a[0] * widths_a[0]
    eps = 1e-12 * max(abs(hi0 - a_origin[0]), 1.0)
    # vectorised over patches; layout per patch: its rows (x), then its columns (y)
    los = np.array([p.spec.lo for p in store.patches], dtype=np.int64).reshape(-1, nd)
    his = np.array([p.spec.hi for p in store.patches], dtype=np.int64).reshape(-1, nd)
    ext = his - los + 1
    per = ext.sum(axis=1)
    poff = np.cumsum(per) - per
    total = int(per.sum())
    W = np.empty(total, np.float64)
    I = np.empty(total, np.int32)
    Dr = np.empty(total, np.int32)
    for ax in range(nd):
        n = ext[:, ax]
        pid = np.repeat(np.arange(len(n)), n)
        t = np.arange(int(n.sum())) - np.repeat(np.cumsum(n) - n, n)
        idx = los[pid, ax] + t
        coord = level_origin[ax] + (idx + 0.5) * widths_f[ax]
        hi = a_origin[ax] + n_a[ax] * widths_a[ax]
        if np.any(coord < a_origin[ax] - eps) or np.any(coord > hi + eps):
            raise OutOfRangeError("interpolation point outside the adjoint domain")
        i0, w = _axis_weights_np(coord, a_origin[ax], widths_a[ax], n_a[ax])
        dry = np.clip(((coord - a_origin[ax]) / widths_a[ax]).astype(int), 0, n_a[ax] - 1)
        pos = poff[pid] + (ext[pid, 0] if ax == 1 else 0) + t
        W[pos] = w
        I[pos] = i0
        Dr[pos] = dry
        # every even-aligned pair along this axis shares its adjoint stencil index
        # (K3 paired row kernel: columns; quad kernel: rows and columns)
        ev = (t % 2 == 0) & (t + 1 < np.repeat(n, n))
        ok = bool(np.all(I[pos[ev]] == I[pos[ev] + 1])) and bool(np.all(n % 2 == 0))
        if ax == 1:
            pairs_ok = ok
        else:
            rows_ok = ok
    offs = np.stack([poff, poff + ext[:, 0]] if nd == 2 else [poff, poff], axis=1).reshape(-1)
    torch = _torch()
    tabs = (torch.from_numpy(W).to("cuda"),
            torch.from_numpy(I).to("cuda"),
            torch.from_numpy(Dr).to("cuda"),
            torch.from_numpy(np.array(offs, dtype=np.int64)).to("cuda"),
            nd == 2 and pairs_ok, nd == 2 and pairs_ok and rows_ok,
            nd == 2 and bool(np.all((W == 0.0) | (W == 1.0))))    # every centre on an adjoint centre
    store._scratch[key] = tabs
    return tabs


K3_ROW_CELLS = 128   # cells per warp of the K3 row-layout kernel (32 lanes x NC)


# K3 window pruning by the window's |snapshot| envelope (AdjFlagArgs.envelope; flags-only calls
# on multi-snapshot windows; flags and counts unchanged).  ADJAMR_FLAG_PRUNE=0 switches it off.
USE_FLAG_PRUNING = os.environ.get("ADJAMR_FLAG_PRUNE", "1") != "0"


def launch_flag(store: LevelStore, ring, ring_shape, a_origin, a_dx, a_dy, level_origin, level_dx, level_dy,
                snap_index, tolerance, adj_wet=None, interp_w=None, want_best=False, stream=None,
                variant=None):
    """K3 on every patch of the store.  ring: (N, m, nxa[, nya]) float64 CUDA
    tensor; snap_index: list of ints (mode 0) or (k, w) pairs (mode 1).
    Returns (flag_bits uint32 tensor, counts (npatch,) int64 tensor,
    best list-of-tensors or None, status tensor)."""
    torch = _torch()
    npatch = len(store.patches)
    mode = 0 if interp_w is None else 1
    # window lists cached on the device (no blocking pageable copy per launch)
    wkey = ("flagwin", tuple(int(k) for k in snap_index),
            None if interp_w is None else tuple(float(x) for x in interp_w))
    cached = store._scratch.get(wkey)
    if cached is None:
        if len(store._scratch) > 256:
            for k in [k for k in store._scratch if isinstance(k, tuple) and k and k[0] == "flagwin"]:
                del store._scratch[k]
        idx = torch.tensor(list(snap_index) if len(snap_index) else [0], dtype=torch.int32, device="cuda")
        w = torch.tensor(list(interp_w) if interp_w is not None and len(interp_w) else [0.0],
                         dtype=torch.float64, device="cuda")
        cached = store._scratch[wkey] = (idx, w)
    idx, w = cached
    bits = store.scratch("flag_bits", max(store.flag_words, 1), torch.int32)
    counts = store.scratch("flag_counts", npatch, torch.int64)
    status = store.scratch("flag_status", 1, torch.int32)
    ncell = [int(np.prod(p.spec.shape)) for p in store.patches]
    best = best_off = None
    if want_best:
        offs = np.concatenate([[0], np.cumsum(ncell)[:-1]]).astype(np.int64)
        best = torch.zeros(int(sum(ncell)), dtype=torch.float64, device="cuda")
        best_off = torch.from_numpy(offs).to("cuda")
    a = _lib.AdjFlagArgs()
    a.q = _ptr(store.buf[store.cur])
    a.aux = _ptr(store.aux)
    a.patches = _ptr(store.table)
    a.ring = _ptr(ring)
    a.adj_wet = _ptr(adj_wet)
    a.snap_index = _ptr(idx)
    a.interp_w = _ptr(w) if mode == 1 else 0
    a.flag_bits = _ptr(bits)
    a.counts = _ptr(counts)
    a.best = _ptr(best)
    a.best_offset = _ptr(best_off)
    a.status = _ptr(status)
    tw, ti, tdry, toff, pairs_ok, quads_ok, direct_ok = flag_axis_tables(store, ring_shape, a_origin, a_dx, a_dy,
                                                                         level_origin, level_dx, level_dy)
    a.axis_w, a.axis_i, a.axis_dry, a.axis_off = _ptr(tw), _ptr(ti), _ptr(tdry), _ptr(toff)
    a.comp_stride = store.plane
    a.aux_stride = store.plane
    a.npatch = npatch
    a.ndim = store.ndim
    a.m = store.m
    a.ghost = store.g
    a.swe = int(store.swe and store.any_dry())   # the forward wet test only matters with dry cells
    a.mode = mode
    a.nidx = len(snap_index)
    a.nxa = ring_shape[0]
    a.nya = ring_shape[1] if store.ndim == 2 else 1
    a.max_cells = max(ncell)
    # row layout: whole 128-cell row segments per warp, interior adjoint corners
    if (store.ndim == 2 and ring_shape[0] >= 2 and ring_shape[1] >= 2
            and bool((store.table_np["ny"] % K3_ROW_CELLS == 0).all())):
        a.layout = (_lib.FLAG_ROWS | (_lib.FLAG_PAIRS if pairs_ok else 0) | (_lib.FLAG_QUADS if quads_ok else 0)
                    | (_lib.FLAG_DIRECT if direct_ok else 0))
        a.max_rows = int(store.table_np["nx"].max())
        a.max_cols = int(store.table_np["ny"].max())
    a.origin_x = level_origin[0]
    a.origin_y = level_origin[1] if store.ndim == 2 else 0.0
    a.dx, a.dy = level_dx, level_dy
    a.a_origin_x = a_origin[0]
    a.a_origin_y = a_origin[1] if store.ndim == 2 else 0.0
    a.a_dx, a.a_dy = a_dx, a_dy
    a.tolerance = tolerance
    a.variant = _lib.VARIANT_EXACT if variant is None else variant
    if not want_best and USE_FLAG_PRUNING and len(snap_index) >= 2:
        # window envelope scratch: cells whose bound cannot reach the tolerance skip the window
        env = store.__dict__.get("_flag_envelope")
        need = 3 * int(np.prod(ring_shape))       # node envelope (k3_bound takes the stencil maximum)
        if env is None or env.numel() < need:
            env = store._flag_envelope = torch.empty(need, dtype=torch.float64, device="cuda")
        a.envelope = _ptr(env)
        t = store.table_np
        nblk = int(((t["nx"].astype(np.int64) // 2) * (t["ny"].astype(np.int64) // 64)).sum())
        work = store.__dict__.get("_flag_work")
        if work is None or work.numel() < 2 + 4 * nblk:
            work = store._flag_work = torch.empty(2 + 4 * max(nblk, 1) + 2, dtype=torch.int32, device="cuda")
        a.work = _ptr(work)
    a.stream = _lib.stream_ptr(stream)
    _lib.check(_lib.lib().adj_flag_adjoint(_lib.C.byref(a)), "adj_flag_adjoint")
    best_list = None
    if want_best:
        best_list = []
        o = 0
        for n in ncell:
            best_list.append(best[o:o + n])
            o += n
    return bits, counts, best_list, status


# ---------------------------------------------------------------------------
# streamed step of a host-resident patch state

def _slab_bounds(NX, g, slabs, ti):
    """Output-row partition o_0 = g < ... < o_S = NX - g on multiples of the
    strip length ti, so every strip starts where the whole-patch step's strips
    start (the fast kernel's last bits depend on a column's place in its
    strip's 3-way unrolled march)."""
    nint = NX - 2 * g
    nstrip = -(-nint // ti)
    S = max(1, min(int(slabs), nstrip))
    cuts = sorted({min(nint, ti * ((nstrip * k) // S)) for k in range(S + 1)})
    return [g + c for c in cuts]


def _fast_tile_shape():
    ni_t, nj_t = _lib.I32(), _lib.I32()
    _lib.check(_lib.lib().adj_step_tile_shape(_lib.VARIANT_FAST, 2, _lib.C.byref(ni_t), _lib.C.byref(nj_t)),
               "adj_step_tile_shape")
    return ni_t.value, nj_t.value


def stream_step(store: LevelStore, host, dt, equation, boundary, level_shape, limiter, slabs=8, wait=True):
    """fill_ghost_physical + the fast step of the single patch of ``store``
    on a state held in host memory ``host`` (m, NX, NY), updated in place.

    Row slabs run on three streams: the H2D copy of slab k+1, the physical
    fill + K1 of slab k and the D2H copy of slab k-1 overlap.  Each slab is a
    virtual patch over the real one (its rows with a g-row halo; x edge bits
    only on the first / last slab), so K1 and the fill run unchanged; the
    halo rows come from the neighbouring chunk, which is copied first.
    Leaves the new state (interior and filled ghosts) in the store's ``cur``.

    ``wait=False``: return with the device-to-host copies in flight (the
    device state is complete for later launches on the current stream; the
    host state is complete after ``stream_finish``).  A following call then
    starts its host-to-device copy of a slab as soon as the copies that
    wrote (or read, on the device) the same rows finished, so consecutive
    steps overlap their two PCIe directions.  Non-finite flags accumulate
    until ``stream_finish``.  Returns None in that mode."""
    torch = _torch()
    p = store.patches[0]
    off, NX, NY, pitch = store.boxes[0]
    g, m = store.g, store.m
    store.edges_table(level_shape)
    edges = int(store.table_np["edges"][0])
    inb = store.cur
    outb = store._free(store.cur, store.ghost_src, -1 if store.old is None else store.old, settle=False)
    ti, tj = _fast_tile_shape()
    ti = store._strip_length(ti, tj)
    o = _slab_bounds(NX, g, slabs, ti)
    S = len(o) - 1
    r = [0] + [o[k] + g for k in range(1, S)] + [NX]      # H2D chunks: slab k needs rows < o[k+1] + g
    d = [0] + o[1:S] + [NX]                                # D2H chunks
    if not hasattr(store, "_streams"):
        store._streams = tuple(torch.cuda.Stream() for _ in range(3))
        store._stream_scratch = torch.zeros(4, dtype=torch.int32, device="cuda")
    s_in, s_cmp, s_out = store._streams
    scratch = store._stream_scratch
    main = torch.cuda.current_stream()
    start = torch.cuda.Event()
    start.record(main)
    for s in (s_in, s_cmp, s_out):
        s.wait_event(start)
    # an unfinished previous call (wait=False): slab k's H2D writes the host rows the previous
    # D2H of slabs k-1..k+1 wrote (and their device rows it read) -> wait for exactly those
    prev = store.__dict__.pop("_stream_pending", None)
    dev_in = store.buf[inb].as_strided((m, NX, NY), (store.plane, pitch, 1), off)
    dev_out = store.buf[outb].as_strided((m, NX, NY), (store.plane, pitch, 1), off)
    # per-slab virtual patch tables and tiles (cached per geometry)
    key = ("stream", tuple(o), edges, ti)
    cached = store._scratch.get(key)
    if cached is None:
        tabs, tiles = [], []
        for k in range(S):
            v = store.table_np[:1].copy()
            v["offset"] = off + (o[k] - g) * pitch
            v["nx"] = o[k + 1] - o[k]
            e = edges & ~(_lib.EDGE_XLO | _lib.EDGE_XHI)
            if k == 0:
                e |= edges & _lib.EDGE_XLO
            if k == S - 1:
                e |= edges & _lib.EDGE_XHI
            v["edges"] = e
            nxv, ny = int(v["nx"][0]), int(v["ny"][0])
            t = [(0, i0, j0, min(ti, nxv - i0), min(tj, ny - j0), 0)
                 for i0 in range(0, nxv, ti) for j0 in range(0, ny, tj)]
            tabs.append(_dev_table(v))
            tiles.append((_dev_table(np.array(t, dtype=_lib.TILE_DTYPE)), len(t)))
        cached = (tabs, tiles)
        store._scratch[key] = cached
    tabs, tiles = cached
    system, form, rev = equation.kernel_spec()
    spec = p.spec
    sides = _bc_codes(boundary)
    ev_in = [torch.cuda.Event() for _ in range(S)]
    ev_cmp = [torch.cuda.Event() for _ in range(S)]
    if prev is None or prev[0] != tuple(o):
        if prev is not None:            # other geometry: wait for every pending copy
            for ev in prev[1]:
                s_in.wait_event(ev)
            prev = None
        with torch.cuda.stream(s_cmp):
            if prev is None and not store.__dict__.get("_stream_acc"):
                scratch.zero_()
    ev_out = [torch.cuda.Event() for _ in range(S)]
    for k in range(S):
        with torch.cuda.stream(s_in):
            if prev is not None:
                for j in (k - 1, k, k + 1):
                    if 0 <= j < S:
                        s_in.wait_event(prev[1][j])
            _copy_rows(dev_in, host, r[k], r[k + 1], s_in)
            ev_in[k].record(s_in)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev_in[k])
            a = _lib.AdjPhysArgs()
            a.q = _ptr(store.buf[inb])
            a.patches = _ptr(tabs[k])
            a.comp_stride = store.plane
            a.npatch, a.ndim, a.ghost, a.m = 1, 2, g, m
            for i, code in enumerate(sides):
                a.bc[i] = code
            a.normal_comp[0] = equation.normal_component(0)
            a.normal_comp[1] = equation.normal_component(1)
            a.max_ghost_cells = (o[k + 1] - o[k] + 2 * g) * NY
            a.stream = _lib.stream_ptr(s_cmp)
            _lib.check(_lib.lib().adj_fill_physical(_lib.C.byref(a)), "adj_fill_physical")
            b = _lib.AdjStepArgs()
            b.q_in = _ptr(store.buf[inb])
            b.q_out = _ptr(store.buf[outb])
            b.aux = _ptr(store.aux)
            b.patches = _ptr(tabs[k])
            b.tiles = _ptr(tiles[k][0])
            b.speed_max = _ptr(store.scratch("smax", 2, torch.float64))
            b.nonfinite = _ptr(scratch)
            b.work_counter = _ptr(scratch[2:])
            b.static_speed = _ptr(store.static_speed())
            b.comp_stride = store.plane
            b.aux_stride = store.plane
            b.npatch, b.ntile, b.ndim, b.ghost = 1, tiles[k][1], 2, g
            b.system, b.form, b.reversed = system, form, rev
            b.limiter = _lib.LIMITERS[limiter]
            b.variant = _lib.VARIANT_FAST
            b.flags = _lib.STEP_KEEP_NONFINITE | _lib.STEP_NO_SPEED_OUT | _lib.STEP_COUNTER_ZERO
            if store.any_dry():      # the wet/dry march for every job (no per-job classes on the slabs)
                b.flags |= _lib.STEP_WET_DRY
            b.dt, b.dtdx, b.dtdy, b.gravity = dt, dt / spec.dx, dt / spec.dy, equation.gravity
            b.stream = _lib.stream_ptr(s_cmp)
            _lib.check(_lib.lib().adj_step_level(_lib.C.byref(b)), "adj_step_level")
            # the output keeps the filled ghosts (the reference's step leaves ghosts untouched)
            lo, hi = d[k], d[k + 1]
            dev_out[:, lo:hi, :g].copy_(dev_in[:, lo:hi, :g])
            dev_out[:, lo:hi, NY - g:].copy_(dev_in[:, lo:hi, NY - g:])
            if k == 0:
                dev_out[:, :g].copy_(dev_in[:, :g])
            if k == S - 1:
                dev_out[:, NX - g:].copy_(dev_in[:, NX - g:])
            ev_cmp[k].record(s_cmp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_cmp[k])
            _copy_rows(host, dev_out, d[k], d[k + 1], s_out)
            ev_out[k].record(s_out)
    store.ghost_src = outb
    store.cur = outb
    if not wait:
        main.wait_stream(s_in)
        main.wait_stream(s_cmp)
        store._stream_pending = (tuple(o), ev_out)
        store._stream_acc = True
        return None
    for s in (s_in, s_cmp, s_out):
        main.wait_stream(s)
    s_out.synchronize()
    store._stream_acc = False
    return bool(scratch[0].item())


def _copy_rows(dst, src, lo, hi, stream):
    """Rows [lo, hi) of every component of (m, NX, NY) views whose rows are
    contiguous (the component planes at any stride): one strided copy
    (adj_copy2d_async) instead of one copy per component."""
    if hi <= lo:
        return
    m, _, NY = src.shape
    width = (hi - lo) * NY * 8
    if not (dst.stride(1) == NY and src.stride(1) == NY and dst.stride(2) == 1 and src.stride(2) == 1):
        for c in range(m):
            dst[c, lo:hi].copy_(src[c, lo:hi], non_blocking=True)
        return
    _lib.check(_lib.lib().adj_copy2d_async(dst[0, lo].data_ptr(), dst.stride(0) * 8, src[0, lo].data_ptr(),
                                           src.stride(0) * 8, width, m, _lib.stream_ptr(stream)),
               "adj_copy2d_async")


def stream_finish(store: LevelStore) -> bool:
    """Complete the pending device-to-host copies of ``stream_step(wait=False)``
    calls; returns whether any of those steps produced a non-finite value."""
    torch = _torch()
    pend = store.__dict__.pop("_stream_pending", None)
    if pend is None and not store.__dict__.get("_stream_acc"):
        return False
    s_in, s_cmp, s_out = store._streams
    main = torch.cuda.current_stream()
    for s in (s_in, s_cmp, s_out):
        main.wait_stream(s)
    s_out.synchronize()
    store._stream_acc = False
    bad = bool(store._stream_scratch[0].item())
    store._stream_scratch.zero_()
    return bad
