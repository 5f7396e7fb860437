"""Batch cores with the reference's positional signatures (_core.py:80-336).

Each function takes the same arguments as the numba core it replaces --
``Octree.core_arrays()`` bundle, kernel id, alpha, distance floor, queries,
method knobs, caller-allocated outputs -- and fills the outputs in place.
The arrays may be numpy (host) or torch CUDA tensors; FP32 float arrays select
the precision="f32" path, exactly as the reference's dtype dispatch does.
The work runs in the sm_100a kernels behind include/fastsum_b200.h.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _device as dev
from . import _lib

RR_PAPER_RATIO = 0
RR_FIXED_HALF = 1
RR_DISABLED = 2

__all__ = ["brute_force_batch", "barnes_hut_batch", "telescoping_batch", "stochastic_batch",
           "stochastic_moments_batch", "RR_PAPER_RATIO", "RR_FIXED_HALF", "RR_DISABLED"]


def _is_f32(a) -> bool:
    t = dev.torch()
    if isinstance(a, t.Tensor):
        return a.dtype == t.float32
    return np.asarray(a).dtype == np.float32


def _dev_f64(a):
    return dev.to_device(a, dev.torch().float64) if isinstance(a, dev.torch().Tensor) else \
        dev.to_device(np.asarray(a, dtype=np.float64))


def _write_back(dst, src_tensor):
    t = dev.torch()
    if isinstance(dst, t.Tensor):
        dst.copy_(src_tensor)
    else:
        dst[...] = src_tensor.cpu().numpy().astype(dst.dtype, copy=False)


def _sp():
    return C.c_void_p(dev.stream_ptr())


def _vp(x):
    return C.c_void_p(dev.ptr(x))


_TREE_CACHE: dict = {}


def _tree_for(core11):
    """Device tree for a core-array bundle (cached by array identity for reuse)."""
    key = tuple(id(a) for a in core11)
    hit = _TREE_CACHE.get(key)
    if hit is not None and all(r() is a for r, a in zip(hit[0], core11)):
        return hit[1]
    from .octree import _upload_core_arrays
    d = _upload_core_arrays(core11)
    import weakref
    refs = []
    for a in core11:
        try:
            refs.append(weakref.ref(a))
        except TypeError:
            refs = None
            break
    if refs is not None:
        if len(_TREE_CACHE) > 8:
            _TREE_CACHE.clear()
        _TREE_CACHE[key] = (refs, d)
    return d


def brute_force_batch(kid, alpha, dfloor, pts, ms, queries, out):
    """_core.py:80-98."""
    f32 = _is_f32(pts)
    p, m_, q = _dev_f64(pts), _dev_f64(ms), _dev_f64(queries)
    n = q.shape[0]
    c = m_.shape[1] if m_.dim() == 2 else 1
    t = dev.torch()
    res = dev.empty(n, t.float32 if f32 else t.float64)
    _lib.check(_lib.lib().fsb_brute_force_batch(int(kid), float(alpha), float(dfloor),
                                                1 if f32 else 0, _vp(p), _vp(m_), p.shape[0], c,
                                                _vp(q), n, _vp(res), _sp()))
    _write_back(out, res)


def barnes_hut_batch(bbox_min, diam, agg_mass, com, child_start, child_count, child_index,
                     begin, end, pts, ms, kid, alpha, dfloor, queries, beta, stack_cap, out,
                     visited):
    """_core.py:101-129 (stack_cap is accepted for signature parity; traversal is stackless)."""
    core = (bbox_min, diam, agg_mass, com, child_start, child_count, child_index, begin, end,
            pts, ms)
    f32 = _is_f32(diam)
    d = _tree_for(core)
    q = _dev_f64(queries)
    n = q.shape[0]
    t = dev.torch()
    res = dev.empty(n, t.float32 if f32 else t.float64)
    vis = dev.empty(n, t.int64)
    _lib.check(_lib.lib().fsb_barnes_hut_batch(C.c_void_p(d.handle), int(kid), float(alpha),
                                               float(dfloor), 1 if f32 else 0, _vp(q), n, None,
                                               float(beta), _vp(res), _vp(vis), _sp()))
    _write_back(out, res)
    _write_back(visited, vis)


def telescoping_batch(bbox_min, diam, agg_mass, com, child_start, child_count, child_index,
                      begin, end, pts, ms, kid, alpha, dfloor, queries, out, visited):
    """_core.py:132-156."""
    core = (bbox_min, diam, agg_mass, com, child_start, child_count, child_index, begin, end,
            pts, ms)
    f32 = _is_f32(diam)
    d = _tree_for(core)
    q = _dev_f64(queries)
    n = q.shape[0]
    t = dev.torch()
    res = dev.empty(n, t.float32 if f32 else t.float64)
    vis = dev.empty(n, t.int64)
    _lib.check(_lib.lib().fsb_telescoping_batch(C.c_void_p(d.handle), int(kid), float(alpha),
                                                float(dfloor), 1 if f32 else 0, _vp(q), n,
                                                _vp(res), _vp(vis), _sp()))
    _write_back(out, res)
    _write_back(visited, vis)


def stochastic_batch(bbox_min, diam, agg_mass, com, child_start, child_count, child_index,
                     begin, end, pts, ms, kid, alpha, dfloor, queries, n_samples, rr_mode, seed,
                     query_offset, out, visited, path_steps, path_count):
    """_core.py:215-267."""
    core = (bbox_min, diam, agg_mass, com, child_start, child_count, child_index, begin, end,
            pts, ms)
    f32 = _is_f32(diam)
    d = _tree_for(core)
    q = _dev_f64(queries)
    n = q.shape[0]
    t = dev.torch()
    res = dev.empty(n, t.float32 if f32 else t.float64)
    vis, st, pc = (dev.empty(n, t.int64) for _ in range(3))
    _lib.check(_lib.lib().fsb_stochastic_batch(
        C.c_void_p(d.handle), int(kid), float(alpha), float(dfloor), 1 if f32 else 0, _vp(q), n,
        None, int(n_samples), int(rr_mode), int(seed) & ((1 << 64) - 1), int(query_offset),
        _vp(res), _vp(vis), _vp(st), _vp(pc), _sp()))
    _write_back(out, res)
    _write_back(visited, vis)
    _write_back(path_steps, st)
    _write_back(path_count, pc)


def stochastic_moments_batch(bbox_min, diam, agg_mass, com, child_start, child_count,
                             child_index, begin, end, pts, ms, kid, alpha, dfloor, queries,
                             n_reps, rr_mode, seed, mean_out, var_out):
    """_core.py:270-336: mean / population variance of n_reps single-sample estimates."""
    core = (bbox_min, diam, agg_mass, com, child_start, child_count, child_index, begin, end,
            pts, ms)
    d = _tree_for(core)
    q = _dev_f64(queries)
    n = q.shape[0]
    t = dev.torch()
    mean = dev.empty(n, t.float64)
    var = dev.empty(n, t.float64)
    _lib.check(_lib.lib().fsb_stochastic_moments_batch(
        C.c_void_p(d.handle), int(kid), float(alpha), float(dfloor), _vp(q), n, int(n_reps),
        int(rr_mode), int(seed) & ((1 << 64) - 1), _vp(mean), _vp(var), _sp()))
    _write_back(mean_out, mean)
    _write_back(var_out, var)


def rr_probability(ratio_parent, ratio_child, mode):
    """_core.py:32-41 (scalar)."""
    if mode == RR_FIXED_HALF:
        return 0.5
    if mode == RR_DISABLED:
        return 1.0
    num = ratio_parent if ratio_parent > 1.0 else 1.0
    den = ratio_child if ratio_child > 1e-12 else 1e-12
    p = num / den
    return p if p < 1.0 else 1.0
