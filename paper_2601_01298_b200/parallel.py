"""Multi-GPU sharding of the hot path.

* Selection groups (layer, KV-head) are independent: rank r owns a contiguous
  block of groups and runs the whole k-round greedy loop locally -- no
  collective during selection.  The single exchange step is an all-gather of
  each rank's landmark rows / scores / K / V so every GPU holds the full
  synapse (NCCL over NVLink; gloo in the CPU tests).
* Decode shards by agent: rank r owns a contiguous block of agents and
  attends against its local synapse replica -- no per-step exchange.
"""
from __future__ import annotations

from typing import Sequence, Tuple

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Balanced contiguous [begin, end) block of n items for `rank` of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def all_gather_groups(local: Sequence[torch.Tensor], n_total: int, group=None) -> list:
    """All-gather per-group tensors sharded by shard_range along dim 0.

    Every tensor in `local` has shape [n_local, ...]; returns tensors of shape
    [n_total, ...] ordered by group id.  Shards are padded to the largest
    shard so a single fixed-size all_gather per tensor suffices.
    """
    world = dist.get_world_size(group)
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    max_n = max(e - b for b, e in sizes)
    out = []
    for t in local:
        pad_shape = (max_n,) + tuple(t.shape[1:])
        padded = torch.zeros(pad_shape, dtype=t.dtype, device=t.device)
        padded[: t.shape[0]] = t
        bufs = [torch.empty_like(padded) for _ in range(world)]
        dist.all_gather(bufs, padded, group=group)
        out.append(torch.cat([bufs[r][: e - b] for r, (b, e) in enumerate(sizes)], dim=0))
    return out
