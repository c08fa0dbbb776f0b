"""World-size-2 gloo test of the N>1 host logic (replica aggregation and the
cell-balanced patch partition) on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1511_03645_b200.replicas import aggregate, partition
    ms, cells = aggregate(10.0 + rank, 1000 * (rank + 1))
    parts = partition([5, 9, 1, 7, 3, 3], world)
    results[rank] = (ms, cells, parts)
    dist.destroy_process_group()


def test_replica_aggregation_gloo_world2():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        res = mgr.dict()
        mp.spawn(_worker, args=(world, port, res), nprocs=world, join=True)
        out = dict(res)
    for r in range(world):
        ms, cells, parts = out[r]
        assert ms == 11.0 and cells == 3000
        assert sorted(sum(parts, [])) == list(range(6))
        assert parts == out[0][2]
    loads = [sum([5, 9, 1, 7, 3, 3][k] for k in p) for p in out[0][2]]
    assert abs(loads[0] - loads[1]) <= 2


def test_aggregate_without_group_is_identity():
    from paper_1511_03645_b200.replicas import aggregate
    assert aggregate(3.5, 7) == (3.5, 7)
