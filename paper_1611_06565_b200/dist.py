"""Multi-GPU plumbing for the batch-sharded layer.

Tiles and samples are independent, so the only shared state is the
transformed filter bank U (read-only): rank 0 runs the filter transform and
U is broadcast once over NCCL (NVLink); each rank then convolves its own batch
slice with no per-forward communication.  When the batch is smaller than the
number of GPUs the output channels are split as well (grid_shard: each rank
transforms its own kernel slice g[k_lo:k_hi] and convolves the full x of its
samples; no reduction).  Timing is the max over ranks.
These helpers are pure torch.distributed calls (nccl on GPUs, gloo in the CPU
tests); no arithmetic of the method lives here.
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def shard_range(batch: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) sample range of `rank` for a global `batch`
    (strong scaling); remainders go to the lowest ranks."""
    base, rem = divmod(batch, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def grid_shape(batch: int, K: int, world: int) -> Tuple[int, int]:
    """(pb, pk) with pb * pk = world: batch shards first (pb = the largest
    divisor of world that is <= batch), output channels split over the rest
    (SURVEY.md 8(e) K-split, 8(f) NEXT-3: batch < GPUs).  Outputs stay sharded
    and no reduction is needed: y[b, k] depends on all of x[b] and on g[k]
    only."""
    if batch < 1 or K < 1 or world < 1:
        raise ValueError("batch, K, world >= 1")
    pb = max(d for d in range(1, world + 1) if world % d == 0 and d <= batch)
    pk = world // pb
    if pk > K:
        raise ValueError("world %d > batch shards %d x K %d" % (world, pb, K))
    return pb, pk


def grid_shard(batch: int, K: int, rank: int, world: int) -> Tuple[int, int, int, int]:
    """[b_lo, b_hi) x [k_lo, k_hi) of `rank` on the (batch x K) grid of
    grid_shape; rank = ib * pk + ik."""
    pb, pk = grid_shape(batch, K, world)
    ib, ik = divmod(rank, pk)
    b_lo, b_hi = shard_range(batch, ib, pb)
    k_lo, k_hi = shard_range(K, ik, pk)
    return b_lo, b_hi, k_lo, k_hi


def gather_outputs(y_local: torch.Tensor, batch: int, K: int, group=None) -> torch.Tensor:
    """Assemble the full y [batch][K][...] from every rank's grid shard (for
    verification only; the forward itself needs no exchange)."""
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if world == 1:
        return y_local
    pb, pk = grid_shape(batch, K, world)
    spatial = tuple(y_local.shape[2:])
    # pad every shard to the largest shard shape so all_gather sees equal sizes
    bmax = -(-batch // pb)
    kmax = -(-K // pk)
    buf = torch.zeros((bmax, kmax) + spatial, dtype=y_local.dtype, device=y_local.device)
    buf[:y_local.shape[0], :y_local.shape[1]] = y_local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    y = torch.empty((batch, K) + spatial, dtype=y_local.dtype, device=y_local.device)
    for r in range(world):
        b_lo, b_hi, k_lo, k_hi = grid_shard(batch, K, r, world)
        y[b_lo:b_hi, k_lo:k_hi] = parts[r][:b_hi - b_lo, :k_hi - k_lo]
    return y


def broadcast_filter(u: torch.Tensor, src: int = 0, group=None) -> None:
    """One broadcast of the transformed filter buffer (U_hi | U_lo) from `src`."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(u, src=src, group=group)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """max of a per-rank scalar (device-timed milliseconds) over all ranks."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def barrier(group=None, device=None) -> None:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if device is not None and dist.get_backend(group) == "nccl":
            dist.barrier(group=group, device_ids=[torch.device(device).index])
        else:
            dist.barrier(group=group)
