"""Sharded uniform level on CPU: slab decomposition, and the
product's halo exchange over a gloo process group (world 2 and 3) with the
oracle's physical fill and step (solver.py:125-146, 442-512) as the compute.
Every rank's interior after K steps must equal the unsharded run's rows
bitwise, with wall and outflow sides and a heterogeneous medium."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import adjamr_oracle as O
from paper_1511_03645_b200.sharded import slab_bounds

G = 2
NX, NY = 23, 17
BC = {"xlo": "wall", "xhi": "outflow", "ylo": "outflow", "yhi": "wall"}
NORMAL = (1, 2)       # acoustics: u normal to x, v normal to y
DX, DY = 0.1, 0.12
STEPS = 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = np.random.default_rng(7)
    shape = (NX + 2 * G, NY + 2 * G)
    rho = rng.uniform(0.8, 1.6, shape)
    bulk = rng.uniform(0.5, 4.0, shape)
    c = np.sqrt(bulk / rho)
    aux = np.stack([c, rho * c, rho, bulk])
    q = rng.standard_normal((3,) + shape)
    dt = 0.8 * min(DX, DY) / c.max()
    return q, aux, dt


def _global_run():
    q, aux, dt = _problem()
    edges = {k: True for k in BC}
    for _ in range(STEPS):
        q = O.fill_physical(q, G, edges, BC, NORMAL)
        q, _ = O.step_2d(q, aux, dt, DX, DY, O.AC2D)
    return q


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1511_03645_b200.sharded import DistTransport, exchange_x_halos
    q, aux, dt = _problem()
    x0, x1 = slab_bounds(NX, world, rank)
    ql = np.array(q[:, x0:x1 + 2 * G], copy=True)
    al = np.array(aux[:, x0:x1 + 2 * G], copy=True)
    nxl = x1 - x0
    has_lo, has_hi = rank > 0, rank < world - 1
    edges = {"xlo": not has_lo, "xhi": not has_hi, "ylo": True, "yhi": True}
    tr = DistTransport(rank, world)
    for _ in range(STEPS):
        ql = O.fill_physical(ql, G, edges, BC, NORMAL)
        t = torch.from_numpy(np.ascontiguousarray(ql)).reshape(-1)
        plane = ql.shape[1] * ql.shape[2]
        exchange_x_halos(t, 3, plane, 0, ql.shape[2], nxl, G, tr, has_lo, has_hi)
        ql = t.reshape(ql.shape).numpy().copy()
        ql, _ = O.step_2d(ql, al, dt, DX, DY, O.AC2D)
    results[rank] = (x0, x1, ql[:, G:-G, G:-G].copy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exchange_gloo_bitwise(world):
    port = _free_port()
    with mp.Manager() as mgr:
        res = mgr.dict()
        mp.spawn(_worker, args=(world, port, res), nprocs=world, join=True)
        out = dict(res)
    ref = _global_run()[:, G:-G, G:-G]
    rows = []
    for r in range(world):
        x0, x1, qi = out[r]
        assert np.array_equal(qi, ref[:, x0:x1]), f"rank {r} differs"
        rows.append((x0, x1))
    assert rows[0][0] == 0 and rows[-1][1] == NX
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))


@pytest.mark.parametrize("nx,world", [(10, 1), (10, 3), (4096, 8), (7, 7)])
def test_slab_bounds_partition(nx, world):
    b = [slab_bounds(nx, world, r) for r in range(world)]
    assert b[0][0] == 0 and b[-1][1] == nx
    assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
    sizes = [x1 - x0 for x0, x1 in b]
    assert max(sizes) - min(sizes) <= 1


def test_slab_bounds_rejects_bad_args():
    with pytest.raises(ValueError):
        slab_bounds(3, 4, 0)
    with pytest.raises(ValueError):
        slab_bounds(8, 2, 2)
