"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

Covers what bench.py does across ranks on the B200 box: the U broadcast from
rank 0 (one collective per weight set), batch sharding, and the max-over-ranks
timing reduction.  The GPU kernels themselves are exercised by -m gpu tests.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_06565_b200.dist import broadcast_filter, max_over_ranks, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # U broadcast: rank 0 holds the transformed filters, others garbage
        u = torch.arange(1000, dtype=torch.float32) * 0.5 if rank == 0 else torch.full((1000,), -7.0)
        broadcast_filter(u, src=0)
        ok_bcast = bool(torch.equal(u, torch.arange(1000, dtype=torch.float32) * 0.5))
        # timing: every rank reports its own ms, all get the max
        m = max_over_ranks(1.5 + rank)
        # strong-scaling shards cover the batch exactly once
        lo, hi = shard_range(7, rank, world)
        q.put((rank, ok_bcast, m, lo, hi))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] for r in res), "broadcast did not deliver rank 0's U"
    assert all(r[2] == 2.5 for r in res), "max over ranks"
    covered = [i for r in sorted(res, key=lambda r: r[3]) for i in range(r[3], r[4])]
    assert covered == list(range(7))


@pytest.mark.parametrize("batch,world", [(32, 1), (32, 8), (7, 3), (1, 2), (16, 4)])
def test_shard_range_partition(batch, world):
    got = [i for r in range(world) for i in range(*shard_range(batch, r, world))]
    assert got == list(range(batch))
    sizes = [shard_range(batch, r, world)[1] - shard_range(batch, r, world)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1
