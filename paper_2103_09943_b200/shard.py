"""Multi-GPU work partitioning of the blind solve: one process per GPU.

The hot path shards naturally and needs no data-path collective:

* by spectral channel (config C3): every rank repeats the per-scene setup (spectral weights,
  TGV kernel fit, intensity normalisation over all bands -- deterministic, so every rank gets
  bit-identical kernels) and reconstructs its contiguous block of bands;
* by scene (config C4, and replicas of C1/C2): every rank solves its block of scenes.

The only communication is gathering the results on rank 0 (``gather_blocks``), which uses
``torch.distributed`` (NCCL for CUDA tensors, gloo for CPU tensors in the tests). The solver
is injected, so the same plumbing runs the GPU path (``fbmp.blind_subset`` /
``fbmp.blind_batch``) and, in the CPU tests, the oracle.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np


def partition(n_items: int, world: int, rank: int) -> range:
    """Contiguous, balanced block of ``n_items`` for ``rank`` (the first n % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def gather_blocks(local: np.ndarray, counts: Sequence[int], group=None, device=None):
    """Concatenate every rank's leading-axis block (sizes ``counts``) on rank 0.

    ``local`` has shape (counts[rank], ...). Returns the concatenation on rank 0, None elsewhere.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mx = max(counts)
    tail = tuple(local.shape[1:])
    buf = torch.zeros((mx,) + tail, dtype=torch.float64, device=device)
    if counts[rank]:
        buf[: counts[rank]] = torch.from_numpy(np.ascontiguousarray(local)).to(buf.device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if rank != 0:
        return None
    return np.concatenate([parts[r][: counts[r]].cpu().numpy() for r in range(world)], axis=0)


def blind_channels_sharded(n_bands: int, solve_subset: Callable[[int, int], np.ndarray], group=None, device=None):
    """Channel-sharded blind solve: ``solve_subset(ch0, nch)`` returns (nch, H, W) on this rank."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world > n_bands:
        raise ValueError("channel sharding needs at least one band per rank")
    mine = partition(n_bands, world, rank)
    counts = [len(partition(n_bands, world, r)) for r in range(world)]
    return gather_blocks(solve_subset(mine.start, len(mine)), counts, group, device)


def blind_scenes_sharded(n_scenes: int, solve_scenes: Callable[[range], np.ndarray], group=None, device=None):
    """Scene-sharded solve: ``solve_scenes(range)`` returns (len(range), N, H, W) on this rank."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = partition(n_scenes, world, rank)
    counts = [len(partition(n_scenes, world, r)) for r in range(world)]
    return gather_blocks(solve_scenes(mine), counts, group, device)
