"""Multi-GPU plumbing for the batch-sharded layer.

Tiles and samples are independent, so the only shared state is the
transformed filter bank U (read-only): rank 0 runs the filter transform and
U is broadcast once over NCCL (NVLink); each rank then convolves its own batch
slice with no per-forward communication.  Timing is the max over ranks.
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
