"""Multi-GPU plumbing for the bench: one process per GPU, independent
replicas of the level, device time reduced as the max over
ranks and work summed.  Also a deterministic cell-balanced partition of a
level's patches across ranks, for sharded flagging / stepping."""
from __future__ import annotations

import numpy as np


def aggregate(ms: float, cells: int, device=None):
    """(max over ranks of ms, sum over ranks of cells); identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(ms), int(cells)
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    c = torch.tensor([cells], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return float(t.item()), int(c.item())


def partition(cell_counts, world: int) -> list[list[int]]:
    """Greedy longest-processing-time split of patch indices over ranks so
    each rank gets about the same number of cells; deterministic."""
    order = sorted(range(len(cell_counts)), key=lambda k: (-int(cell_counts[k]), k))
    load = np.zeros(world, dtype=np.int64)
    out = [[] for _ in range(world)]
    for k in order:
        r = int(np.argmin(load))
        out[r].append(k)
        load[r] += int(cell_counts[k])
    return [sorted(o) for o in out]
