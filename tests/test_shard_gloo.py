"""Multi-rank host logic of the batch-sharded path on CPU with gloo, world_size 2."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2101_05917_b200 import shard


def test_shard_range_partitions():
    for n in (1, 7, 8, 64):
        for w in (1, 2, 3, 8):
            got = [shard.shard_range(n, w, r) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [h - l for l, h in got]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 5
    lo, hi = shard.shard_range(n, world, rank)
    local = torch.arange(lo, hi, dtype=torch.float64)[:, None] * torch.ones(1, 3, dtype=torch.float64)
    full = shard.gather_rows(local, world)
    t = shard.max_over_ranks(10.0 + rank, world)
    out[rank] = (full.tolist(), t)
    dist.destroy_process_group()


def test_gather_and_max_over_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        full, t = out[r]
        assert full == [[float(i)] * 3 for i in range(5)]
        assert t == 11.0


def test_shared_youngs_ref_is_batch_max():
    assert shard.shared_youngs_ref([1.0, 3.0, 2.0]) == 3.0
