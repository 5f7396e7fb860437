"""ctypes front end of the C oracle (TEST INFRASTRUCTURE ONLY).

Mirrors the positional signatures of the reference's numba cores
(``/root/reference/pkg/src/fastsum/_core.py:80-336``) and of
``build_tree`` (``octree.py:118-239``) so parity tests read like the
reference's own.  Only ``tests/``, ``__graft_entry__.smoke()`` and the CPU
legs of ``bench.py`` may import this module; the product package never does.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int64)


class _TreeOut(C.Structure):
    _fields_ = [("num_nodes", C.c_int64)] + [
        (k, _D) for k in ("bbox_min", "bbox_max", "diameter", "agg_mass", "agg_weight", "com")
    ] + [
        (k, _I) for k in ("child_start", "child_count", "child_index", "begin", "end",
                          "depth", "perm")
    ]


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH)
                < os.path.getmtime(os.path.join(_HERE, "fastsum_oracle.c"))):
            build()
        L = C.CDLL(_LIB_PATH)
        L.or_stream_key.restype = C.c_uint64
        L.or_stream_key.argtypes = [C.c_uint64] * 5
        L.or_uniform_draw.restype = C.c_double
        L.or_uniform_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.or_rr_probability.restype = C.c_double
        L.or_rr_probability.argtypes = [C.c_double, C.c_double, C.c_int]
        L.or_np_sum.restype = C.c_double
        L.or_np_sum.argtypes = [_D, C.c_int64]
        L.or_build_tree.restype = C.c_int
        L.or_build_tree.argtypes = [_D, _D, _D, C.c_int64, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(_TreeOut)]
        L.or_free_tree.argtypes = [C.POINTER(_TreeOut)]
        _lib = L
    return _lib


def _dp(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(_D)


def _ip(a):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_I)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _tree_args(core11):
    (_bbox_min, diam, agg_mass, com, cs, cc, ci, b, e, pts, ms) = core11
    agg_mass = _f64(agg_mass)
    c = agg_mass.shape[1] if agg_mass.ndim == 2 else 1
    keep = [_f64(diam), agg_mass, _f64(com), _i64(cs), _i64(cc), _i64(ci), _i64(b),
            _i64(e), _f64(pts), _f64(ms)]
    args = [_dp(keep[0]), _dp(keep[1]), _dp(keep[2]), _ip(keep[3]), _ip(keep[4]),
            _ip(keep[5]), _ip(keep[6]), _ip(keep[7]), _dp(keep[8]), _dp(keep[9]),
            C.c_int64(keep[6].shape[0]), C.c_int(c)]
    return keep, args


# ------------------------------------------------------------------ cores
def brute_force_batch(kid, alpha, dfloor, pts, ms, queries, out):
    """_core.py:80-98."""
    pts, ms, q = _f64(pts), _f64(ms), _f64(queries)
    c = ms.shape[1] if ms.ndim == 2 else 1
    res = np.zeros(q.shape[0])
    fn = lib().or_brute_force_batch
    fn(C.c_int(kid), C.c_double(alpha), C.c_double(dfloor), _dp(pts), _dp(ms),
       C.c_int64(pts.shape[0]), C.c_int(c), _dp(q), C.c_int64(q.shape[0]), _dp(res))
    out[:] = res


def barnes_hut_batch(*args):
    """_core.py:101-129; args = core11 + (kid, alpha, dfloor, queries, beta, stack_cap, out, visited)."""
    core11, (kid, alpha, dfloor, queries, beta, stack_cap, out, visited) = args[:11], args[11:]
    keep, targs = _tree_args(core11)
    q = _f64(queries)
    res = np.zeros(q.shape[0])
    vis = np.zeros(q.shape[0], dtype=np.int64)
    lib().or_barnes_hut_batch(*targs, C.c_int(kid), C.c_double(alpha), C.c_double(dfloor),
                              _dp(q), C.c_int64(q.shape[0]), C.c_double(beta),
                              C.c_int64(stack_cap), _dp(res), _ip(vis))
    out[:] = res
    visited[:] = vis


def telescoping_batch(*args):
    """_core.py:132-156."""
    core11, (kid, alpha, dfloor, queries, out, visited) = args[:11], args[11:]
    keep, targs = _tree_args(core11)
    q = _f64(queries)
    res = np.zeros(q.shape[0])
    vis = np.zeros(q.shape[0], dtype=np.int64)
    lib().or_telescoping_batch(*targs, C.c_int(kid), C.c_double(alpha), C.c_double(dfloor),
                               _dp(q), C.c_int64(q.shape[0]), _dp(res), _ip(vis))
    out[:] = res
    visited[:] = vis


def stochastic_batch(*args):
    """_core.py:215-267."""
    core11 = args[:11]
    (kid, alpha, dfloor, queries, n_samples, rr_mode, seed, query_offset, out, visited,
     path_steps, path_count) = args[11:]
    keep, targs = _tree_args(core11)
    q = _f64(queries)
    n = q.shape[0]
    res = np.zeros(n)
    vis, st, pc = (np.zeros(n, dtype=np.int64) for _ in range(3))
    lib().or_stochastic_batch(*targs, C.c_int(kid), C.c_double(alpha), C.c_double(dfloor),
                              _dp(q), C.c_int64(n), C.c_int64(n_samples), C.c_int(rr_mode),
                              C.c_uint64(int(seed)), C.c_int64(query_offset), _dp(res),
                              _ip(vis), _ip(st), _ip(pc))
    out[:] = res
    visited[:] = vis
    path_steps[:] = st
    path_count[:] = pc


def stochastic_ex_batch(*args, keys=None, variant=0):
    """stochastic_batch plus the paper's options (not in the reference): query i draws
    from the streams of index keys[i] (None: i + query_offset), variant 1 = Alg. 2;
    args = core11 + (kid, alpha, dfloor, queries, n_samples, rr_mode, seed, query_offset,
    out, visited, path_steps, path_count)."""
    core11 = args[:11]
    (kid, alpha, dfloor, queries, n_samples, rr_mode, seed, query_offset, out, visited,
     path_steps, path_count) = args[11:]
    keep, targs = _tree_args(core11)
    q = _f64(queries)
    n = q.shape[0]
    k = None if keys is None else np.ascontiguousarray(keys, dtype=np.uint64)
    res = np.zeros(n)
    vis, st, pc = (np.zeros(n, dtype=np.int64) for _ in range(3))
    lib().or_stochastic_ex_batch(*targs, C.c_int(kid), C.c_double(alpha), C.c_double(dfloor),
                                 _dp(q), C.c_int64(n), C.c_int64(n_samples), C.c_int(rr_mode),
                                 C.c_uint64(int(seed)), C.c_int64(query_offset),
                                 None if k is None else k.ctypes.data_as(C.c_void_p),
                                 C.c_int(variant), _dp(res), _ip(vis), _ip(st), _ip(pc))
    out[:] = res
    visited[:] = vis
    path_steps[:] = st
    path_count[:] = pc


def barnes_hut_vote_batch(*args):
    """Warp-voting BH (not in the reference): groups of 32 consecutive
    positions of `order`; args = core11 + (kid, alpha, dfloor, queries, order, beta, out,
    visited)."""
    core11, (kid, alpha, dfloor, queries, order, beta, out, visited) = args[:11], args[11:]
    keep, targs = _tree_args(core11)
    q = _f64(queries)
    o = None if order is None else np.ascontiguousarray(order, dtype=np.int32)
    res = np.zeros(q.shape[0])
    vis = np.zeros(q.shape[0], dtype=np.int64)
    lib().or_barnes_hut_vote_batch(*targs, C.c_int(kid), C.c_double(alpha), C.c_double(dfloor),
                                   _dp(q), C.c_int64(q.shape[0]),
                                   None if o is None else o.ctypes.data_as(C.c_void_p),
                                   C.c_double(beta), _dp(res), _ip(vis))
    out[:] = res
    visited[:] = vis


def stochastic_moments_batch(*args):
    """_core.py:270-336."""
    core11 = args[:11]
    (kid, alpha, dfloor, queries, n_reps, rr_mode, seed, mean_out, var_out) = args[11:]
    keep, targs = _tree_args(core11)
    q = _f64(queries)
    n = q.shape[0]
    mean = np.zeros(n)
    var = np.zeros(n)
    lib().or_stochastic_moments_batch(*targs, C.c_int(kid), C.c_double(alpha),
                                      C.c_double(dfloor), _dp(q), C.c_int64(n),
                                      C.c_int64(n_reps), C.c_int(rr_mode),
                                      C.c_uint64(int(seed)), _dp(mean), _dp(var))
    mean_out[:] = mean
    var_out[:] = var


# ------------------------------------------------------------------- tree
def build_tree(positions, masses, weights, branching_per_dim=2, max_depth=32) -> dict:
    """octree.py:118-239; returns the 16 per-node/per-point arrays by slot name."""
    pos = _f64(positions)
    ms = _f64(masses)
    if ms.ndim == 1:
        ms = ms[:, None]
    w = _f64(weights)
    m, c = pos.shape[0], ms.shape[1]
    t = _TreeOut()
    rc = lib().or_build_tree(_dp(pos), _dp(ms), _dp(w), C.c_int64(m), C.c_int(c),
                             C.c_int(branching_per_dim), C.c_int(max_depth), C.byref(t))
    if rc != 0:
        raise ValueError("oracle build_tree: bad arguments")
    n = t.num_nodes

    def cp(ptr, count, dt, shape):
        if count == 0:
            return np.zeros(shape, dtype=dt)
        return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dt, copy=True).reshape(shape)

    out = dict(
        bbox_min=cp(t.bbox_min, 3 * n, np.float64, (n, 3)),
        bbox_max=cp(t.bbox_max, 3 * n, np.float64, (n, 3)),
        diameter=cp(t.diameter, n, np.float64, (n,)),
        aggregate_mass=cp(t.agg_mass, c * n, np.float64, (n, c)),
        aggregate_weight=cp(t.agg_weight, n, np.float64, (n,)),
        center_of_mass=cp(t.com, 3 * n, np.float64, (n, 3)),
        child_start=cp(t.child_start, n, np.int64, (n,)),
        child_count=cp(t.child_count, n, np.int64, (n,)),
        child_index=cp(t.child_index, n - 1, np.int64, (n - 1,)),
        begin=cp(t.begin, n, np.int64, (n,)),
        end=cp(t.end, n, np.int64, (n,)),
        depth=cp(t.depth, n, np.int64, (n,)),
        permuted_indices=cp(t.perm, m, np.int64, (m,)),
    )
    lib().or_free_tree(C.byref(t))
    perm = out["permuted_indices"]
    out["points"] = np.ascontiguousarray(pos[perm])
    out["masses"] = np.ascontiguousarray(ms[perm])
    out["weights"] = np.ascontiguousarray(w[perm])
    out["branching_per_dim"] = int(branching_per_dim)
    out["max_depth"] = int(max_depth)
    return out


def core_arrays(t: dict):
    """Octree.core_arrays order, octree.py:110-115."""
    return (t["bbox_min"], t["diameter"], t["aggregate_mass"], t["center_of_mass"],
            t["child_start"], t["child_count"], t["child_index"], t["begin"], t["end"],
            t["points"], t["masses"])


# -------------------------------------------------------------------- rng
def stream_key(seed, qi, sub, sample, stream) -> int:
    return int(lib().or_stream_key(int(seed), int(qi), int(sub), int(sample), int(stream)))


def uniform_draw(key, counter) -> float:
    return float(lib().or_uniform_draw(int(key), int(counter)))


def draws(seed, qi, sub, sample, stream, count) -> np.ndarray:
    out = np.zeros(count)
    fn = lib().or_draws
    fn.argtypes = [C.c_uint64] * 5 + [C.c_int64, _D]
    fn(int(seed), int(qi), int(sub), int(sample), int(stream), count, _dp(out))
    return out


def rr_probability(rp, rc, mode) -> float:
    return float(lib().or_rr_probability(rp, rc, mode))


def np_sum(a) -> float:
    a = _f64(a)
    return float(lib().or_np_sum(_dp(a), a.shape[0]))


def shuffle_order(n, seed, query_offset=0):
    """The warp-shared mode's evaluation order (restates fsb_shuffle_order)."""
    perm = np.zeros(int(n), dtype=np.int32)
    lib().or_shuffle_order(C.c_int64(n), C.c_uint64(int(seed)), C.c_int64(query_offset),
                           perm.ctypes.data_as(C.c_void_p))
    return perm


def shared_keys(n, seed, query_offset=0, group_log2=5):
    """keys[i] of stochastic_ex_batch for the warp-shared mode: the group index of the
    position query i takes in shuffle_order (positions offset by query_offset)."""
    order = shuffle_order(n, seed, query_offset).astype(np.int64)
    keys = np.zeros(int(n), dtype=np.uint64)
    keys[order] = ((np.arange(n) + query_offset) >> group_log2).astype(np.uint64)
    return keys
