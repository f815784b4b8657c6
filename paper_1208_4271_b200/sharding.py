"""Multi-GPU sharding of a pair batch: pairs are independent, so
each rank scores its share of the condensed PairSequence order
(analysis.cpp:66-81) on its own GPU with a full replica of the (small) input,
and the only collective is one final gather of the per-rank result slices --
nothing crosses ranks on the data path.  Results are bit-identical for any
world size (each pair's arithmetic depends only on its own inputs).

Two assignments:
  * "range"  -- one contiguous range per rank (the weak-scaling bench: every
    c1 pair costs about the same);
  * "cyclic" -- chunks of `chunk` pairs dealt round-robin (SURVEY 8e balance:
    pair cost varies 10-100x between independent and functional pairs, e.g.
    c4, so a contiguous split can leave one rank with the expensive block).
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


def shard_chunks(total: int, world: int, rank: int, chunk: int) -> list[tuple[int, int]]:
    """Round-robin chunks of [0, total): the (first, count) windows of `rank`."""
    if world < 1 or not 0 <= rank < world or chunk < 1:
        raise ValueError("shard_chunks: bad world/rank/chunk")
    return [(f, min(chunk, total - f)) for f in range(rank * chunk, total, world * chunk)]


def gather_cyclic(local: dict, total: int, chunk: int, dist, device=None, stats=None) -> dict:
    """All-gather round-robin chunk results (each rank's chunks concatenated in
    order) and re-interleave them into the condensed order on every rank."""
    import torch
    world = dist.get_world_size()
    sizes = [sum(c for _, c in shard_chunks(total, world, r, chunk)) for r in range(world)]
    width = max(sizes)
    out = {}
    for key in stats or sorted(local):
        v = torch.as_tensor(np.ascontiguousarray(local[key]), dtype=torch.float64)
        if device is not None:
            v = v.to(device)
        buf = torch.zeros(width, dtype=torch.float64, device=v.device)
        buf[: v.numel()] = v
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
        full = np.empty(total, dtype=np.float64)
        for r, part in enumerate(parts):
            host = part.cpu().numpy()
            pos = 0
            for first, cnt in shard_chunks(total, world, r, chunk):
                full[first:first + cnt] = host[pos:pos + cnt]
                pos += cnt
        out[key] = full
    return out


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
                  device=None, strategy: str = "range", chunk: int = 4096) -> dict:
    """Run `score_range(first, count)` over this rank's share and gather.  With
    dist=None (or world size 1) this is just score_range(0, total).  With
    strategy="cyclic" the scorer is called once per chunk window (a GPU scorer
    passes reuse_vars=True after its first window)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return score_range(0, total)
    world, rank = dist.get_world_size(), dist.get_rank()
    if strategy == "range":
        first, count = shard_range(total, world, rank)
        return gather_condensed(score_range(first, count), total, dist, device)
    if strategy != "cyclic":
        raise ValueError(f"score_sharded: unknown strategy {strategy!r}")
    parts = [score_range(f, c) for f, c in shard_chunks(total, world, rank, chunk)]
    # the statistic names, from rank 0 (a rank may own no chunk)
    box = [None]
    if rank == 0:
        box[0] = sorted(parts[0] if parts else score_range(0, 0))
    dist.broadcast_object_list(box, src=0)
    keys = box[0]
    local = {k: np.concatenate([p[k] for p in parts]) if parts else np.empty(0) for k in keys}
    return gather_cyclic(local, total, chunk, dist, device, keys)
