"""Multi-GPU sharding of a pair batch: pairs are independent, so
each rank scores a contiguous range of the condensed PairSequence order
(analysis.cpp:66-81) on its own GPU with a full replica of the (small) input,
and the only collective is one final gather of the per-rank result slices --
nothing crosses ranks on the data path.  Results are bit-identical for any
world size (each pair's arithmetic depends only on its own inputs).
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split of [0, total): (first, count) of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad world/rank")
    first = rank * total // world
    return first, (rank + 1) * total // world - first


def gather_condensed(local: dict, total: int, dist, device=None, stats=None) -> dict | None:
    """All-gather each rank's slice of every statistic into the full condensed
    arrays (rank order == condensed order).  Slices are padded to a common
    length so one all_gather per statistic suffices (NCCL or gloo).  Returns
    the full arrays on every rank."""
    import torch
    world = dist.get_world_size()
    width = (total + world - 1) // world
    out = {}
    for key in stats or sorted(local):
        v = torch.as_tensor(np.ascontiguousarray(local[key]), dtype=torch.float64)
        if device is not None:
            v = v.to(device)
        buf = torch.zeros(width, dtype=torch.float64, device=v.device)
        buf[: v.numel()] = v
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
        pieces = []
        for r, part in enumerate(parts):
            _, cnt = shard_range(total, world, r)
            pieces.append(part[:cnt].cpu().numpy())
        out[key] = np.concatenate(pieces)
    return out


def score_sharded(score_range: Callable[[int, int], dict], total: int, dist=None,
                  device=None) -> dict:
    """Run `score_range(first, count)` on this rank's shard and gather.  With
    dist=None (or world size 1) this is just score_range(0, total)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return score_range(0, total)
    first, count = shard_range(total, dist.get_world_size(), dist.get_rank())
    local = score_range(first, count)
    return gather_condensed(local, total, dist, device)
