"""Query-slab sharding across ranks.

Queries are independent and every stochastic draw is keyed on the *global*
query index (stochastic_batch's ``query_offset``, reference _core.py:219,258),
so rank r evaluates the contiguous slab [r*N/P, (r+1)*N/P) with
query_offset = slab start and the gathered field is identical to a
single-process evaluation.  The tree is a replica per rank (the GPU build is
deterministic, so every rank builds the same bits); results are gathered with
one all_gather -- the only collective on this path.
"""

from __future__ import annotations

import numpy as np

__all__ = ["slab", "gather_slabs", "evaluate_field_sharded"]


def slab(n: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) of rank's contiguous, balanced share of n queries."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_slabs(local, n: int, group=None):
    """All-gather equal-or-ragged slabs (torch tensors, 1-D) into the full (n,) field."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = [slab(n, r, world)[1] - slab(n, r, world)[0] for r in range(world)]
    width = max(sizes)
    pad = torch.zeros(width, dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])


def evaluate_field_sharded(config, sources, kernel, queries, tree=None, group=None):
    """evaluate_field over this rank's slab; returns the gathered values (host numpy)."""
    import torch.distributed as dist
    from .estimators import evaluate_field_device
    from .types import QuerySet
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = len(queries)
    a, b = slab(n, rank, world)
    local = evaluate_field_device(config, sources, kernel, QuerySet(queries.positions[a:b]), tree,
                                  query_offset=a)
    return gather_slabs(local.values, n, group).cpu().numpy()
