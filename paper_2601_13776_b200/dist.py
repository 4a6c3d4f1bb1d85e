"""Multi-GPU plumbing of the hot path (reading R22).

Construction is sharded by layer: every rank creates the plan with its
(rank, world), orthogonalises and composes only the layers it owns, writing
them into its rank-major segment of the kernel buffer (offsets from
``orth_plan_query``).  One all-gather of the segments then gives every rank all
kernels; the forward shards over the batch with no collective.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def gather_kernels(plan, kbuf: torch.Tensor, seg: int, group=None) -> torch.Tensor:
    """All-gather the rank-major segments of ``kbuf`` (length world * seg) in place."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return kbuf
    mine = kbuf[rank * seg:(rank + 1) * seg].clone()
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(kbuf, mine, group=group)
    else:  # gloo: list form
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        kbuf.copy_(torch.cat(parts))
    return kbuf


def batch_shard(n_total: int, rank: int, world: int):
    """[begin, end) of this rank's images (weak scaling uses n_total per rank)."""
    per = (n_total + world - 1) // world
    b = min(n_total, rank * per)
    return b, min(n_total, b + per)
