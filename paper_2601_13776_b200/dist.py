"""Multi-GPU plumbing of the hot path (reading R22).

Construction is sharded by (layer, group) unit, LPT over NS + composition
flops: every rank creates the plan with its (rank, world), orthogonalises and
composes only the units it owns, writing them into its rank-major segment of
the GATHER buffer (``orth_compose_kernel`` with world > 1).  One all-gather of
the equal segments (NCCL over NVLink: in place, no staging copy) gives every
rank every unit; ``orth_kernels_assemble`` (one copy kernel) then lays the
units out as contiguous per-layer kernels for ``orth_conv_forward``.  The
forward shards over the batch with no collective.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def gather_kernels(gbuf: torch.Tensor, seg: int, group=None) -> torch.Tensor:
    """All-gather the rank-major equal segments of ``gbuf`` (length world * seg) in place."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return gbuf
    mine = gbuf[rank * seg:(rank + 1) * seg]
    if dist.get_backend(group) == "nccl":
        # in place: NCCL allows sendbuff == recvbuff + rank * count
        dist.all_gather_into_tensor(gbuf, mine, group=group)
    else:  # gloo: list form
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine.clone(), group=group)
        gbuf.copy_(torch.cat(parts))
    return gbuf


def batch_shard(n_total: int, rank: int, world: int):
    """[begin, end) of this rank's images of a global batch (strong scaling)."""
    per = (n_total + world - 1) // world
    b = min(n_total, rank * per)
    return b, min(n_total, b + per)
