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

from paper_1611_06565_b200.dist import (broadcast_filter, gather_outputs, grid_shape, grid_shard, max_over_ranks,
                                        shard_range)


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
        # batch 1 < 2 ranks: output channels split; the gathered shards
        # rebuild the full y (each rank fills only its own slice)
        yfull = torch.arange(1 * 5 * 3 * 4, dtype=torch.float32).reshape(1, 5, 3, 4)
        b0, b1, k0, k1 = grid_shard(1, 5, rank, world)
        ok_gather = bool(torch.equal(gather_outputs(yfull[b0:b1, k0:k1].clone(), 1, 5), yfull))
        # batch 3 x K 4 over 2 ranks: batch shards, full K each
        b0, b1, k0, k1 = grid_shard(3, 4, rank, world)
        y2 = torch.randn(3, 4, 2, generator=torch.Generator().manual_seed(5))
        ok_gather2 = bool(torch.equal(gather_outputs(y2[b0:b1, k0:k1].clone(), 3, 4), y2))
        q.put((rank, ok_bcast, m, lo, hi, ok_gather, ok_gather2))
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
    assert all(r[5] and r[6] for r in res), "gather of (batch x K) grid shards"


@pytest.mark.parametrize("batch,K,world", [(32, 128, 8), (1, 4, 4), (1, 128, 8), (2, 64, 8), (3, 5, 6), (6, 7, 4)])
def test_grid_shard_partition(batch, K, world):
    pb, pk = grid_shape(batch, K, world)
    assert pb * pk == world and pb <= batch and pk <= K
    if batch >= world:
        assert pk == 1                       # batch sharding whenever it suffices
    cells = []
    for r in range(world):
        b0, b1, k0, k1 = grid_shard(batch, K, r, world)
        assert b1 > b0 and k1 > k0
        cells += [(b, k) for b in range(b0, b1) for k in range(k0, k1)]
    assert sorted(cells) == [(b, k) for b in range(batch) for k in range(K)]


def test_grid_shape_too_many_ranks():
    with pytest.raises(ValueError):
        grid_shape(1, 2, 4)


@pytest.mark.parametrize("batch,world", [(32, 1), (32, 8), (7, 3), (1, 2), (16, 4)])
def test_shard_range_partition(batch, world):
    got = [i for r in range(world) for i in range(*shard_range(batch, r, world))]
    assert got == list(range(batch))
    sizes = [shard_range(batch, r, world)[1] - shard_range(batch, r, world)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1
