"""Query-slab sharding across ranks.

Queries are independent and every stochastic draw is keyed on the *global*
query index (stochastic_batch's ``query_offset``, reference _core.py:219,258),
so rank r evaluates the contiguous slab [r*N/P, (r+1)*N/P) with
query_offset = slab start and the gathered field is identical to a
single-process evaluation (with the paper's warp-shared streams the slab
boundaries are multiples of the 2^16-position shuffle window, so the same holds).
The tree is a replica per rank (the GPU build is
deterministic, so every rank builds the same bits); results are gathered with
one all_gather -- the only collective on this path.
"""

from __future__ import annotations

import numpy as np

__all__ = ["slab", "gather_slabs", "evaluate_field_sharded", "broadcast_tree", "SHUFFLE_WINDOW"]

SHUFFLE_WINDOW = 1 << 16  # positions per window of fsb_shuffle_order (warp-shared mode)


def slab(n: int, rank: int, world: int, align: int = 1) -> tuple[int, int]:
    """[start, stop) of rank's contiguous, balanced share of n queries; with align > 1
    every boundary but the end is a multiple of align (the warp-shared mode's 2^16
    shuffle windows, so slabs evaluate exactly as inside the whole set)."""
    if world < 1 or not 0 <= rank < world or align < 1:
        raise ValueError("bad rank / world size / alignment")

    def cut(r):
        if r >= world:
            return n
        base, extra = divmod(n, world)
        c = r * base + min(r, extra)
        return min(n, (c + align // 2) // align * align) if align > 1 else c

    return cut(rank), cut(rank + 1)


def gather_slabs(local, n: int, group=None, align: int = 1):
    """All-gather equal-or-ragged slabs (torch tensors, 1-D) into the full (n,) field."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = [slab(n, r, world, align)[1] - slab(n, r, world, align)[0] for r in range(world)]
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
    a, b = slab(n, rank, world, SHUFFLE_WINDOW if _shared(config) else 1)
    import torch
    # precision="f32" values of the non-smooth kernels are FP32 results widened to
    # FP64 (the post-transform is the identity): gathered as FP32, 4 B per query
    # (SURVEY 5), and widened after the collective -- the same bits
    narrow = config.precision == "f32" and kernel.kind != "smooth_exp"
    if b > a:
        local = evaluate_field_device(config, sources, kernel, QuerySet(queries.positions[a:b]),
                                      tree, query_offset=a).values
    else:  # more ranks than slabs: this rank contributes nothing
        local = torch.empty(0, dtype=torch.float64, device="cuda")
    if narrow:
        local = local.to(torch.float32)
    full = gather_slabs(local, n, group, SHUFFLE_WINDOW if _shared(config) else 1)
    return full.to(torch.float64).cpu().numpy()


def _shared(config) -> bool:
    return (getattr(config, "method", "") == "stochastic"
            and getattr(config, "rng_sharing", "query") == "warp")


def broadcast_tree(sources, branching_per_dim: int = 2, max_depth: int = 32, src: int = 0,
                   group=None):
    """The tree built once on rank `src` and broadcast (NCCL over NVLink with the nccl
    backend) to every rank -- the alternative to per-rank replica builds.

    Rank `src` builds from `sources` (other ranks may pass None) and exports the ten
    device core arrays (Octree.core_arrays() minus the unused bbox_min) straight into
    device buffers; every other rank receives them and assembles its handle with
    fsb_tree_from_core_arrays (a device-to-device copy; the per-rank packed records are
    rebuilt lazily from them).  Returns an Octree on every rank; the result is
    bit-identical to the source rank's tree.
    """
    import ctypes as C
    import torch
    import torch.distributed as dist
    from . import _device as dev
    from . import _lib
    from .octree import Octree, _DeviceTree, build_tree
    rank = dist.get_rank(group)
    device = torch.device("cuda", torch.cuda.current_device())
    meta = torch.zeros(3, dtype=torch.int64, device=device)
    tree = None
    if rank == src:
        tree = build_tree(sources, branching_per_dim, max_depth)
        d = tree._device_tree()
        meta[:] = torch.tensor([d.num_nodes, d.num_points, d.channels], dtype=torch.int64)
    dist.broadcast(meta, src, group=group)
    n, m, c = (int(v) for v in meta.cpu())
    f64, i64 = torch.float64, torch.int64
    # export order (fsb_tree_export): bbox_min, bbox_max, diameter, aggregate_mass,
    # aggregate_weight, center_of_mass, child_start, child_count, child_index, begin,
    # end, depth, permuted_indices, points, masses, weights
    spec = {2: ((n,), f64), 3: ((n, c), f64), 5: ((n, 3), f64), 6: ((n,), i64), 7: ((n,), i64),
            8: ((max(n - 1, 1),), i64), 9: ((n,), i64), 10: ((n,), i64), 13: ((m, 3), f64),
            14: ((m, c), f64)}
    bufs = {k: torch.empty(shape, dtype=dt, device=device) for k, (shape, dt) in spec.items()}
    if rank == src:
        ptrs = (C.c_void_p * 16)(*[dev.ptr(bufs[k]) if k in bufs else None for k in range(16)])
        _lib.check(_lib.lib().fsb_tree_export(C.c_void_p(tree._device_tree().handle), ptrs,
                                              C.c_void_p(dev.stream_ptr())))
    for k in sorted(bufs):
        dist.broadcast(bufs[k], src, group=group)
    if rank == src:
        return tree
    torch.cuda.synchronize()
    h = C.c_void_p()
    order = (2, 3, 5, 6, 7, 8, 9, 10, 13, 14)
    _lib.check(_lib.lib().fsb_tree_from_core_arrays(
        *[C.c_void_p(dev.ptr(bufs[k])) for k in order], n, m, c, C.byref(h),
        C.c_void_p(dev.stream_ptr())))
    return Octree._from_device(_DeviceTree(h.value), branching_per_dim, max_depth)
