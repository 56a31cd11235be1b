"""Sharding of the search space and the trace batch across GPUs of one node.

One process per GPU (torch.distributed; NCCL on GPUs, gloo on CPU for the
tests).  The search shards the candidate index range into contiguous
blocks; each rank runs K2 on its block and the per-rank winners are
combined with ONE all-reduce of a [world, 3] int64 slot buffer (each rank
writes its own slot: total as raw fp64 bits, index, feasible count; zeros
elsewhere, so the sum is exact), followed by a local lexicographic reduce
(max total, then lowest index) -- the tie rule of planner.py:227.  Trace
replay needs no collective: traces are independent.
"""

from __future__ import annotations

import numpy as np


def shard_range(size: int, rank: int, world: int) -> tuple:
    """Contiguous [lo, hi) block of rank `rank` (blocks differ by <= 1)."""
    return size * rank // world, size * (rank + 1) // world


def pack_slot(world: int, rank: int, total: float, index: int, n_feasible: int) -> np.ndarray:
    buf = np.zeros((world, 3), np.int64)
    buf[rank, 0] = np.float64(total).view(np.int64)
    buf[rank, 1] = index
    buf[rank, 2] = n_feasible
    return buf


def reduce_slots(buf: np.ndarray) -> tuple:
    """Lexicographic reduce of the gathered slots: (total, index, n_feasible)."""
    best_t, best_i = 0.0, -1
    for r in range(buf.shape[0]):
        t = float(np.int64(buf[r, 0]).view(np.float64))
        i = int(buf[r, 1])
        if i >= 0 and (best_i < 0 or t > best_t or (t == best_t and i < best_i)):
            best_t, best_i = t, i
    return best_t, best_i, int(buf[:, 2].sum())


def combine_best(total: float, index: int, n_feasible: int, group=None, device=None, stream=None) -> tuple:
    """All-reduce the per-rank winners (one collective).  `device` is the
    torch device of the buffer (cuda for NCCL, cpu for gloo); `stream` an
    optional torch stream to issue the collective on."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return total, index, n_feasible
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    slot = torch.from_numpy(pack_slot(world, rank, total, index, n_feasible))
    if device is not None:
        slot = slot.to(device)
    if stream is not None:
        stream.wait_stream(torch.cuda.current_stream(slot.device))  # the slot's copy lands first
        with torch.cuda.stream(stream):
            dist.all_reduce(slot, group=group)
            host = slot.cpu().numpy()
    else:
        dist.all_reduce(slot, group=group)
        host = slot.cpu().numpy()
    return reduce_slots(host)


def distributed_search_best(tables, group=None, engine=None, device=None, stream=None) -> tuple:
    """K2 on this rank's shard of the full space + the combine.  Returns
    (total, index, n_feasible) of the whole space on every rank."""
    import torch.distributed as dist

    from .planner import search_best

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(tables.space_size, rank, world)
    total, idx, nfeas, _ms = search_best(tables, lo, hi, engine=engine)
    return combine_best(total, idx, nfeas, group=group, device=device, stream=stream)
