"""fsb_evaluate_field_host through the C ABI with the caller's own output columns.

evaluate_field hands the library one pinned block whose 8-byte columns are
equally spaced, and the host pipeline then moves a slab's columns in one 2-D
copy.  A C-ABI caller may pass any separately allocated (pageable) arrays, or
leave optional columns null; the pipeline then copies column by column.  Both
layouts must give the same bytes, for every method (brute force, BH,
telescoping, stochastic) and slab count; so must pinned and pageable query
arrays (the latter staged by the library's worker threads).  Reference contract:
estimators.py:260-323 (host in, host out; outputs caller-allocated,
estimators.py:273-276).
"""

import ctypes as C

import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_02219_b200 as fs
    return fs


CONFIGS = [
    ("brute_force", dict(precision="f32")),
    ("barnes_hut", dict(beta=2.0, precision="f32")),
    ("barnes_hut", dict(beta=2.0)),
    ("telescoping_exhaustive", dict()),
    ("stochastic", dict(seed=5, precision="f32")),
    ("stochastic", dict(seed=5, precision="f32", rng_sharing="warp")),
    ("stochastic", dict(seed=5)),
]


def _args(fs, cfg, kern, src):
    from paper_2506_02219_b200 import _lib
    from paper_2506_02219_b200.estimators import _RR_CODES, _variant, kernel_id, device_sources
    a = _lib.EvalArgs()
    a.method = _lib.METHOD_CODES[cfg.method]
    a.kid = kernel_id(kern)
    a.alpha, a.dfloor = float(kern.alpha), float(kern.distance_floor)
    a.precision = 1 if cfg.precision == "f32" else 0
    a.beta = float(cfg.beta)
    a.n_samples = int(cfg.samples_per_subdomain)
    a.rr_mode = _RR_CODES[cfg.rr_mode]
    a.seed = int(cfg.seed)
    a.smooth = 0
    a.query_order = 1
    a.rng_group_log2 = 5 if getattr(cfg, "rng_sharing", "query") == "warp" else 0
    a.path_variant = _variant(cfg)
    keep = []
    if cfg.method == "brute_force":
        pts, ms = device_sources(src)[:2]
        keep += [pts, ms]
        from paper_2506_02219_b200 import _device as dev
        a.src_pts, a.src_ms = dev.ptr(pts), dev.ptr(ms)
        a.m, a.c = len(src), src.channel_count
    return a, keep


@pytest.mark.parametrize("method,kw", CONFIGS, ids=lambda x: x if isinstance(x, str) else
                         "-".join(f"{k}={v}" for k, v in sorted(x.items())))
def test_separate_columns_equal_the_pinned_block(fs, method, kw):
    from paper_2506_02219_b200 import _lib
    from paper_2506_02219_b200 import _device as dev
    s = scenes.build_sources(dict(kind="mesh_torus", m=30000, seed=3))
    kern = fs.KernelSpec("coulomb")
    rng = np.random.default_rng(8)
    q = np.ascontiguousarray(rng.uniform(-0.6, 0.6, (300_001, 3)))
    cfg = fs.EstimatorConfig(method, **kw)
    tree = fs.build_tree(s, cfg.resolved_branching)
    L = _lib.lib()
    h = None if method == "brute_force" else C.c_void_p(tree._device_tree().handle)
    for chunks in (1, 3, 8):
        ref = fs.evaluate_field(cfg, s, kern, fs.QuerySet(q), tree=tree, chunks=chunks)
        a, keep = _args(fs, cfg, kern, s)
        n = len(q)
        for with_raw in (True, False):
            # separately allocated pageable columns (no common pitch), some null
            out = dict(values=np.full(n, np.nan), raw=np.full(n, np.nan) if with_raw else None,
                       flagged=np.ones(n, dtype=np.uint8), visited=np.full(n, -1, np.int64),
                       path_steps=np.full(n, -1, np.int64), path_count=np.full(n, -1, np.int64))
            ptr = {k: (C.c_void_p(v.ctypes.data) if v is not None else None) for k, v in out.items()}
            _lib.check(L.fsb_evaluate_field_host(
                h, C.byref(a), q.ctypes.data_as(C.c_void_p), n, ptr["values"], ptr["raw"],
                ptr["flagged"], ptr["visited"], ptr["path_steps"], ptr["path_count"], chunks,
                C.c_void_p(dev.stream_ptr())))
            np.testing.assert_array_equal(out["values"], ref.values, err_msg=f"{chunks}")
            if with_raw:
                np.testing.assert_array_equal(out["raw"], ref.raw)
            np.testing.assert_array_equal(out["flagged"].view(bool), ref.flagged)
            np.testing.assert_array_equal(out["visited"], ref.visited_nodes)
            np.testing.assert_array_equal(out["path_steps"], ref.path_steps)
            np.testing.assert_array_equal(out["path_count"], ref.path_count)
        del keep


@pytest.mark.parametrize("method,kw", [("stochastic", dict(seed=3, precision="f32")),
                                       ("stochastic", dict(seed=3)),
                                       ("barnes_hut", dict(beta=1.5))],
                         ids=["sto-f32", "sto-f64", "bh-f64"])
def test_pageable_and_pinned_queries_give_the_same_bytes(fs, method, kw):
    """Pinned queries are copied to the device directly; pageable ones are first
    staged into page-locked memory slab by slab by the library's worker threads.
    Both must give identical results for any slab count."""
    import torch
    s = scenes.build_sources(dict(kind="mesh_torus", m=30000, seed=3))
    kern = fs.KernelSpec("coulomb")
    q = np.ascontiguousarray(np.random.default_rng(9).uniform(-0.6, 0.6, (400_003, 3)))
    pinned = torch.empty(q.shape, dtype=torch.float64, pin_memory=True)
    pinned.numpy()[:] = q
    cfg = fs.EstimatorConfig(method, **kw)
    tree = fs.build_tree(s, cfg.resolved_branching)
    for chunks in (1, 5):
        a = fs.evaluate_field(cfg, s, kern, fs.QuerySet(q), tree=tree, chunks=chunks)
        b = fs.evaluate_field(cfg, s, kern, fs.QuerySet(pinned.numpy()), tree=tree, chunks=chunks)
        for f in ("values", "raw", "flagged", "visited_nodes", "path_steps", "path_count"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f"{f} {chunks}")
