"""The four field evaluators (reference: estimators.py) on the B200 kernels.

``evaluate_field`` keeps the reference's signature, validation order and
FieldResult contract (estimators.py:260-323); the batch work is one call
through the C ABI per method, with inputs uploaded once and the tree kept
device-resident.  The scalar sampling primitives (``contribution_swap``,
``sample_path_index``, ``russian_roulette_prob``, ``walk_path_sample``) are
host utilities mirroring the reference one query at a time, as in the
reference they exist for tests and interactive use.
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _core
from . import _device as dev
from . import _lib
from .kernels import contribution_rows, kernel_id, node_contribution
from .octree import Octree, TreeNode, build_tree, device_sources, far_field_ratio
from .rng import RngStreams
from .types import EstimatorConfig, KernelSpec, QuerySet, SourceSet

__all__ = ["FieldResult", "PathSampleState", "brute_force", "barnes_hut",
           "telescoping_exhaustive", "path_sample_estimate", "russian_roulette_prob",
           "contribution_swap", "sample_path_index", "walk_path_sample", "evaluate_field",
           "evaluate_field_device"]

_RR_CODES = {"paper_ratio": _core.RR_PAPER_RATIO, "fixed_half": _core.RR_FIXED_HALF,
             "disabled": _core.RR_DISABLED}


@dataclass(frozen=True)
class FieldResult:
    """Per-query estimates plus instrumentation (estimators.py:45-64)."""

    values: np.ndarray
    raw: np.ndarray
    flagged: np.ndarray
    visited_nodes: np.ndarray
    path_steps: np.ndarray
    path_count: np.ndarray
    method: str

    @property
    def flagged_count(self) -> int:
        return int(self.flagged.sum())


@dataclass
class PathSampleState:
    subdomain: int
    point_index: int
    depth: int
    p_agg: float
    p_rr_cumulative: float
    running_sum: float


def _worker_count() -> int:
    """FASTSUM_THREADS parsing (estimators.py:79-88); GPU work ignores it, kept for API parity."""
    raw = os.environ.get("FASTSUM_THREADS", "0")
    try:
        n = int(raw)
    except ValueError:
        n = 0
    return _thread_cap() if n <= 0 else min(n, _thread_cap())


def _thread_cap() -> int:
    """The host thread pool size the reference caps at (numba.config.NUMBA_NUM_THREADS:
    the NUMBA_NUM_THREADS variable, else the CPUs this process may run on)."""
    try:
        v = int(os.environ.get("NUMBA_NUM_THREADS", ""))
        if v > 0:
            return v
    except ValueError:
        pass
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def _check_channels(sources: SourceSet, kernel: KernelSpec) -> None:
    if sources.channel_count != kernel.channel_count:
        raise ValueError(f"kernel {kernel.kind!r} needs {kernel.channel_count} mass channels, "
                         f"sources have {sources.channel_count}")


def _stack_cap(tree: Octree) -> int:
    return int(tree.max_depth + 2) * int(tree.branching_per_dim) ** 3 + 8


def _vp(x):
    return C.c_void_p(dev.ptr(x))


def _sp():
    return C.c_void_p(dev.stream_ptr())


class DeviceField:
    """Device-resident outputs of one evaluation (torch CUDA tensors)."""

    __slots__ = ("values", "raw", "flagged", "visited", "path_steps", "path_count", "method")

    def __init__(self, **kw):
        for k, v in kw.items():
            setattr(self, k, v)

    def to_host(self) -> FieldResult:
        torch = dev.torch()
        # pinned (cached) host buffers, async copies, one synchronisation
        host = []
        for x in (self.values, self.raw, self.flagged, self.visited, self.path_steps,
                  self.path_count):
            h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
            h.copy_(x, non_blocking=True)
            host.append(h)
        torch.cuda.current_stream().synchronize()
        return FieldResult(values=host[0].numpy(), raw=host[1].numpy(),
                           flagged=host[2].numpy().view(bool), visited_nodes=host[3].numpy(),
                           path_steps=host[4].numpy(), path_count=host[5].numpy(),
                           method=self.method)


def evaluate_field_device(config: EstimatorConfig, sources: SourceSet, kernel: KernelSpec,
                          queries, tree: Octree | None = None, *, source_buffers=None,
                          query_order: bool = True, query_offset: int = 0) -> DeviceField:
    """evaluate_field without the final device->host copy.

    ``queries`` may be a QuerySet or an (N,3) float64 CUDA tensor (already
    resident); results stay on the device.  query_offset keys the RNG streams
    on global query indices (stochastic_batch's ``query_offset``, _core.py:219),
    which is how query slabs are sharded across ranks without changing results.
    """
    _check_channels(sources, kernel)
    L = _lib.lib()
    torch = dev.torch()
    q = queries if isinstance(queries, torch.Tensor) else dev.to_device(queries.positions)
    n = q.shape[0]
    f32 = config.precision == "f32"
    prec = 1 if f32 else 0
    raw = dev.empty(n, torch.float32 if f32 else torch.float64)
    visited = dev.empty(n, torch.int64)
    # the stochastic kernels write every counter; the other methods report none
    if config.method == "stochastic":
        steps, count = dev.empty(n, torch.int64), dev.empty(n, torch.int64)
    else:
        steps, count = dev.zeros(n, torch.int64), dev.zeros(n, torch.int64)
    kid = kernel_id(kernel)
    alpha, dfloor = float(kernel.alpha), float(kernel.distance_floor)
    if config.method == "brute_force":
        if source_buffers is None:
            source_buffers = device_sources(sources)[:2]
        pts, ms = source_buffers
        _lib.check(L.fsb_brute_force_batch(kid, alpha, dfloor, prec, _vp(pts), _vp(ms),
                                           len(sources), sources.channel_count, _vp(q), n,
                                           _vp(raw), _sp()))
        visited.fill_(len(sources))
    else:
        if tree is None:
            tree = _tree_for(sources, config.resolved_branching, config.max_depth)
        elif tree.branching_per_dim != config.resolved_branching:
            raise ValueError("prebuilt tree branching factor does not match config")
        h = C.c_void_p(tree._device_tree().handle)
        perm = None
        # Morton order of the queries pays for BH (warp-coherent traversal); the
        # stochastic kernel's node set is query-independent (dense part) or
        # keyed on the sampled point (walks), so it takes queries as given
        if query_order and config.method == "barnes_hut" and n > 1:
            perm = dev.empty(n, torch.int32)
            _lib.check(L.fsb_query_order(_vp(q), n, _vp(perm), _sp()))
        if config.method == "barnes_hut":
            fn = (L.fsb_barnes_hut_vote_batch if getattr(config, "bh_warp_vote", False)
                  else L.fsb_barnes_hut_batch)
            _lib.check(fn(h, kid, alpha, dfloor, prec, _vp(q), n, _vp(perm), float(config.beta),
                          _vp(raw), _vp(visited), _sp()))
        elif config.method == "telescoping_exhaustive":
            _lib.check(L.fsb_telescoping_batch(h, kid, alpha, dfloor, prec, _vp(q), n, _vp(raw),
                                               _vp(visited), _sp()))
        elif (getattr(config, "rng_sharing", "query") == "warp"
              or _variant(config) != 0):
            # the paper's options (fsb_stochastic_batch_ex): shared streams over a
            # shuffled order (32 consecutive positions per stream), Alg. 2 walk
            # (FSB_FLAG_SHUFFLED = 2: fsb_shuffle_order's permutation, computed in-kernel)
            shared = getattr(config, "rng_sharing", "query") == "warp"
            _lib.check(L.fsb_stochastic_batch_ex(
                h, kid, alpha, dfloor, prec, _vp(q), n, None,
                int(config.samples_per_subdomain), _RR_CODES[config.rr_mode],
                int(config.seed) & ((1 << 64) - 1), int(query_offset), 5 if shared else 0,
                _variant(config) | (2 if shared else 0),
                _vp(raw), _vp(visited), _vp(steps), _vp(count), _sp()))
        else:
            _lib.check(L.fsb_stochastic_batch(
                h, kid, alpha, dfloor, prec, _vp(q), n, _vp(perm),
                int(config.samples_per_subdomain), _RR_CODES[config.rr_mode],
                int(config.seed) & ((1 << 64) - 1), int(query_offset), _vp(raw), _vp(visited),
                _vp(steps), _vp(count), _sp()))
    values = dev.empty(n, torch.float64)
    raw64 = dev.empty(n, torch.float64)
    flagged = dev.empty(n, torch.uint8)
    _lib.check(L.fsb_post_transform(_vp(raw), 1 if f32 else 0, n,
                                    1 if kernel.kind == "smooth_exp" else 0, alpha, _vp(values),
                                    _vp(raw64), _vp(flagged), _sp()))
    return DeviceField(values=values, raw=raw64, flagged=flagged, visited=visited,
                       path_steps=steps, path_count=count, method=config.method)


_TREE_CACHE: dict = {}  # the last trees built for an immutable SourceSet, per device
_TREE_LOCK = threading.Lock()


def _tree_for(sources: SourceSet, branching: int, max_depth: int):
    """build_tree for calls without a prebuilt tree, reusing the device tree of the
    most recent SourceSet (immutable: SourceSet owns frozen copies of its arrays,
    so the tree is the same bits): repeated evaluate_field calls on one scene pay
    the build once.  Only the latest SourceSet is kept (weakly): its trees are
    freed with it or when another scene is evaluated.  Keyed on the current CUDA
    device too (a device tree is only valid on the device that built it), and
    locked so two host threads never build or evict concurrently."""
    key = (dev.torch().cuda.current_device(), branching, max_depth)
    with _TREE_LOCK:
        ref = _TREE_CACHE.get("src")
        if ref is not None and ref() is sources and key in _TREE_CACHE["trees"]:
            return _TREE_CACHE["trees"][key]
        if ref is None or ref() is not sources:
            _TREE_CACHE.clear()
            _TREE_CACHE["src"] = weakref.ref(
                sources, lambda r: _TREE_CACHE.clear() if _TREE_CACHE.get("src") is r else None)
            _TREE_CACHE["trees"] = {}
        tree = build_tree(sources, branching, max_depth)
        _TREE_CACHE["trees"][key] = tree
        return tree


def _variant(config) -> int:
    """fsb path variant: 0 the reference's walk, 1 the paper's Alg. 2."""
    return 1 if getattr(config, "path_order", "swap_then_roulette") == "roulette_then_swap" else 0


_PINNED: list = []  # (tensor, ndarray) pinned output blocks, reused once unreferenced
_PINNED_LOCK = threading.Lock()


def _pinned_block(nbytes: int):
    """(data pointer, uint8 ndarray) of a pinned host block of >= nbytes.  Result
    arrays are numpy views of the block's ndarray (their .base chain ends there),
    so a block whose ndarray has no other referrers is free and is reused:
    page-locking fresh memory costs tens of ms per call.  Under a lock: the
    caller's reference exists before another thread can test the block."""
    torch = dev.torch()
    with _PINNED_LOCK:
        for t, mem in _PINNED:
            # referrers: the pool tuple, the loop variable, getrefcount's argument
            if sys.getrefcount(mem) <= 3 and mem.nbytes >= nbytes:
                return t.data_ptr(), mem
        t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        entry = (t, t.numpy())
        _PINNED.append(entry)
        if len(_PINNED) > 4:  # keep the pool small: drop the oldest free block
            for i, (_, old) in enumerate(_PINNED[:-1]):
                if sys.getrefcount(old) <= 3:
                    del _PINNED[i]
                    break
        return entry[0].data_ptr(), entry[1]


def _pipeline_chunks(n: int, config=None) -> int:
    """Slabs for the host pipeline: enough to overlap PCIe with compute, each
    slab still several waves of 148 SMs x 4 blocks x 256 queries (C4, 10^6
    queries: 6 slabs 0.89 ms, 8 slabs 0.92, 4 slabs 1.00; tools/e2e_chunks.py).
    Barnes-Hut takes fewer (tools/e2e_f64.py, C4): the load-balanced FP32 kernel
    synchronises with the host between its work-splitting rounds, so slabs
    serialise (beta 6.4: 4.7 ms in one slab, 20.7 in six), and each FP64 slab pays
    its own longest-chunk tail (beta 2: 2.58 ms in three slabs, 2.75 in six)."""
    cap = 6
    if config is not None and config.method == "barnes_hut":
        cap = 1 if config.precision == "f32" else 3
    return int(max(1, min(cap, n // 160_000)))


def evaluate_field(config: EstimatorConfig, sources: SourceSet, kernel: KernelSpec,
                   queries: QuerySet, tree: Octree | None = None, *,
                   chunks: int | None = None, query_offset: int = 0) -> FieldResult:
    """estimators.py:260-323: dispatch on config.method, then post-transform.

    Host queries in, host results out, through fsb_evaluate_field_host: slabs
    of queries are copied, evaluated and copied back on overlapping streams
    (results are independent of the slab count).  Outputs land in pinned host
    buffers returned as numpy arrays.  ``query_offset`` (an extension; the
    reference keys on 0..n-1) keys the stochastic RNG on global query indices so
    a slab of a larger query set evaluates exactly as inside the whole set.
    """
    _check_channels(sources, kernel)
    L = _lib.lib()
    torch = dev.torch()
    q = np.ascontiguousarray(queries.positions, dtype=np.float64)
    n = q.shape[0]
    args = _lib.EvalArgs()
    args.method = _lib.METHOD_CODES[config.method]
    args.kid = kernel_id(kernel)
    args.alpha, args.dfloor = float(kernel.alpha), float(kernel.distance_floor)
    args.precision = 1 if config.precision == "f32" else 0
    args.beta = float(config.beta)
    args.n_samples = int(config.samples_per_subdomain)
    args.rr_mode = _RR_CODES[config.rr_mode]
    args.seed = int(config.seed) & ((1 << 64) - 1)
    args.query_offset = int(query_offset)
    args.smooth = 1 if kernel.kind == "smooth_exp" else 0
    args.query_order = 1
    # the paper's warp-shared streams (shuffled windows, fsb_shuffle_order)
    args.rng_group_log2 = 5 if (config.method == "stochastic"
                                and getattr(config, "rng_sharing", "query") == "warp") else 0
    args.bh_warp_vote = 1 if getattr(config, "bh_warp_vote", False) else 0
    args.path_variant = _variant(config)
    h = None
    keep = []
    if config.method == "brute_force":
        pts, ms = device_sources(sources)[:2]
        keep += [pts, ms]
        args.src_pts, args.src_ms = dev.ptr(pts), dev.ptr(ms)
        args.m, args.c = len(sources), sources.channel_count
    else:
        if tree is None:
            tree = _tree_for(sources, config.resolved_branching, config.max_depth)
        elif tree.branching_per_dim != config.resolved_branching:
            raise ValueError("prebuilt tree branching factor does not match config")
        h = C.c_void_p(tree._device_tree().handle)
    # one pinned block for all outputs: 8-byte columns values, visited, path_steps,
    # raw, path_count, then the flags (the library copies values and the int32
    # counters across PCIe; raw, path_count and the flags are written on the host)
    base, mem = _pinned_block(41 * n + 8)
    ptrs = [base + 8 * n * k for k in range(5)] + [base + 40 * n]
    _lib.check(L.fsb_evaluate_field_host(
        h, C.byref(args), q.ctypes.data_as(C.c_void_p), n,
        C.c_void_p(ptrs[0]), C.c_void_p(ptrs[3]), C.c_void_p(ptrs[5]), C.c_void_p(ptrs[1]),
        C.c_void_p(ptrs[2]), C.c_void_p(ptrs[4]),
        int(chunks if chunks is not None else _pipeline_chunks(n, config)), _sp()))
    cols = [mem[8 * n * k: 8 * n * (k + 1)] for k in range(5)]
    return FieldResult(values=cols[0].view(np.float64), raw=cols[3].view(np.float64),
                       flagged=mem[40 * n: 41 * n].view(bool),
                       visited_nodes=cols[1].view(np.int64), path_steps=cols[2].view(np.int64),
                       path_count=cols[4].view(np.int64), method=config.method)


# ------------------------------------------------------- single-query wrappers
def _one(config, sources, kernel, q, tree=None, query_offset=0) -> float:
    qs = QuerySet(np.asarray(q, dtype=np.float64).reshape(1, 3))
    r = evaluate_field_device(config, sources, kernel, qs, tree, query_order=False,
                              query_offset=query_offset)
    return float(r.raw.cpu().numpy()[0])


def brute_force(sources: SourceSet, kernel: KernelSpec, q) -> float:
    _check_channels(sources, kernel)
    return _one(EstimatorConfig("brute_force"), sources, kernel, q)


def barnes_hut(tree: Octree, sources: SourceSet, kernel: KernelSpec, q, beta: float) -> float:
    if not beta > 0:
        raise ValueError("beta must be positive")
    _check_channels(sources, kernel)
    cfg = EstimatorConfig("barnes_hut", beta=float(beta),
                          branching_per_dim=tree.branching_per_dim, max_depth=tree.max_depth)
    return _one(cfg, sources, kernel, q, tree)


def telescoping_exhaustive(tree: Octree, sources: SourceSet, kernel: KernelSpec, q) -> float:
    _check_channels(sources, kernel)
    cfg = EstimatorConfig("telescoping_exhaustive", branching_per_dim=tree.branching_per_dim,
                          max_depth=tree.max_depth)
    return _one(cfg, sources, kernel, q, tree)


def path_sample_estimate(tree: Octree, sources: SourceSet, kernel: KernelSpec, q,
                         samples_per_subdomain: int, rr_mode: str = "paper_ratio", seed: int = 0,
                         query_index: int = 0) -> float:
    if samples_per_subdomain < 1:
        raise ValueError("samples_per_subdomain must be >= 1")
    _check_channels(sources, kernel)
    cfg = EstimatorConfig("stochastic", samples_per_subdomain=int(samples_per_subdomain),
                          rr_mode=rr_mode, seed=seed, branching_per_dim=tree.branching_per_dim,
                          max_depth=tree.max_depth)
    return _one(cfg, sources, kernel, q, tree, query_offset=int(query_index))


# ------------------------------------------------------ scalar sampling helpers
def russian_roulette_prob(ratio_parent: float, ratio_child: float,
                          mode: str = "paper_ratio") -> float:
    if ratio_parent < 0 or ratio_child < 0:
        raise ValueError("far field ratios must be non-negative")
    return float(_core.rr_probability(float(ratio_parent), float(ratio_child), _RR_CODES[mode]))


def _leaf_exact_term(kernel: KernelSpec, tree: Octree, i: int, q) -> float:
    b, e = int(tree.begin[i]), int(tree.end[i])
    if tree.child_count[i] == 0 and e - b > 1:
        kid = kernel_id(kernel)
        acc = 0.0
        for j in range(b, e):
            acc += contribution_rows(kid, kernel.alpha, kernel.distance_floor, tree.masses, j,
                                     tree.points[j, 0], tree.points[j, 1], tree.points[j, 2],
                                     q[0], q[1], q[2])
        return acc
    return node_contribution(kernel, tree.node(i), q)


def contribution_swap(kernel: KernelSpec, tree: Octree, node, q) -> float:
    """Children's terms minus the parent's aggregate term (estimators.py:163-178)."""
    if isinstance(node, TreeNode):
        node = node.index
    if tree.child_count[node] == 0:
        raise ValueError("contribution_swap requires an internal node")
    q = np.asarray(q, dtype=np.float64)
    total = 0.0
    s = int(tree.child_start[node])
    for t in range(int(tree.child_count[node])):
        total += _leaf_exact_term(kernel, tree, int(tree.child_index[s + t]), q)
    return total - node_contribution(kernel, tree.node(node), q)


def sample_path_index(stream, tree: Octree, node) -> int:
    if isinstance(node, TreeNode):
        node = node.index
    b, e = int(tree.begin[node]), int(tree.end[node])
    u = stream.next_float()
    j = b + int(u * (e - b))
    if j >= e:
        j = e - 1
    return int(tree.permuted_indices[j])


def walk_path_sample(tree: Octree, sources: SourceSet, kernel: KernelSpec, q, subdomain: int,
                     subdomain_ordinal: int, sample_ordinal: int, seed: int,
                     rr_mode: str = "paper_ratio", query_index: int = 0):
    """Pure-Python mirror of one path sample (estimators.py:207-253)."""
    q = np.asarray(q, dtype=np.float64)
    streams = RngStreams(seed, query_index, subdomain_ordinal, sample_ordinal)
    b, e = int(tree.begin[subdomain]), int(tree.end[subdomain])
    count_a = e - b
    u0 = streams.index_stream.next_float()
    j = min(b + int(u0 * count_a), e - 1)
    node = subdomain
    prr = 1.0
    resid = 0.0
    k = 0
    yield PathSampleState(subdomain=subdomain, point_index=int(tree.permuted_indices[j]), depth=k,
                          p_agg=1.0, p_rr_cumulative=prr, running_sum=resid)
    while tree.child_count[node] > 0:
        s = int(tree.child_start[node])
        child = -1
        for t in range(int(tree.child_count[node])):
            c = int(tree.child_index[s + t])
            if tree.begin[c] <= j < tree.end[c]:
                child = c
                break
        delta = contribution_swap(kernel, tree, node, q)
        pagg = (tree.end[node] - tree.begin[node]) / count_a
        resid += delta / (pagg * prr)
        p = russian_roulette_prob(far_field_ratio(tree.node(node), q),
                                  far_field_ratio(tree.node(child), q), rr_mode)
        yield PathSampleState(subdomain=subdomain, point_index=int(tree.permuted_indices[j]),
                              depth=k, p_agg=float(pagg), p_rr_cumulative=prr, running_sum=resid)
        if streams.roulette_stream.next_float() >= p:
            return
        prr *= p
        node = child
        k += 1
