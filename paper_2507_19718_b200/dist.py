"""Multi-GPU modes of the cache (north star; the paper runs on one GPU).

One process per GPU.  Mode 0 (data parallel): every rank holds a full replica of all levels,
fits its own shard of the frame's samples, and the library performs ONE NCCL all-reduce (sum)
per gc_fit of the per-level coefficient gradients and level statistics before the identical
AdamW step.  Mode 1 (level-sharded): the library routes each sample / lookup to the rank
group owning its level (gc_level_plan), each group fits only its levels.  SURVEY 8(e);
DESIGN.md "Multi-GPU".  torch.distributed is only plumbing: it carries the 128-byte
ncclUniqueId from rank 0 to the others (any backend, gloo included).
"""
from __future__ import annotations

import torch.distributed as dist

from . import nccl_unique_id


def exchange_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes."""
    rank = dist.get_rank(group)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def attach_data_parallel(cache, group=None, uid: bytes | None = None) -> None:
    """Make `cache` a data-parallel replica of the process group (mode 0)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if uid is None:
        uid = exchange_unique_id(group)
    cache.set_comm(uid, rank, world, 0)


def attach_level_sharded(cache, group=None, uid: bytes | None = None, weights=None) -> None:
    """Make `cache` one rank of a level-sharded cache (mode 1); every later gc_fit / gc_query /
    gc_fit_query / gc_params call on it is collective over the group."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if uid is None:
        uid = exchange_unique_id(group)
    cache.set_level_weights(weights)
    cache.set_comm(uid, rank, world, 1)


def attach_owner_computes(cache, group=None, uid: bytes | None = None) -> None:
    """Make `cache` one rank of a spatial owner-computes cache (mode 2, next row f4): samples and
    lookups go to the owner of their cell column, only boundary Gaussians' gradients and rows
    are exchanged.  Collective like mode 1."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if uid is None:
        uid = exchange_unique_id(group)
    cache.set_comm(uid, rank, world, 2)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of n samples for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)
