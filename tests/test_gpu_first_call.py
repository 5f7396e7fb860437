"""First use of a fresh tree through the host pipeline (fsb_evaluate_field_host).

The evaluators pack their node records lazily on first use (fs_pack.cu
ensure_*).  The host pipeline runs odd slabs on a second compute stream, so a
record published before its pack kernel finished would be read half-written by
slab 1.  These tests evaluate 10^6 queries in 8 slabs on a tree that has never
been evaluated, and compare with a device-resident evaluation on an
independently built (bit-identical, F4) tree: bytes must be equal, every time.
Reference contract: estimators.py:260-323 (host in, host out), SURVEY 8(b)
threading (re-entrant across streams and host threads).
"""

import threading

import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu

N_QUERIES = 1_000_000
CASES = [  # (method, precision, rng_sharing)
    ("barnes_hut", "f64", "query"),
    ("stochastic", "f64", "query"),
    ("stochastic", "f32", "query"),
    ("stochastic", "f32", "warp"),
    ("barnes_hut", "f32", "query"),
]


@pytest.fixture(scope="module")
def fs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_02219_b200 as fs
    return fs


@pytest.fixture(scope="module")
def scene(fs):
    s = scenes.build_sources(dict(kind="mesh_torus", m=2 ** 22, seed=31))  # C4 size
    rng = np.random.default_rng(12)
    q = np.column_stack([rng.uniform(-0.5, 0.5, (N_QUERIES, 2)), np.full(N_QUERIES, 0.03)])
    return s, fs.QuerySet(q)


def _cfg(fs, method, prec, sharing):
    if method == "barnes_hut":
        return fs.EstimatorConfig("barnes_hut", beta=2.0, precision=prec)
    return fs.EstimatorConfig("stochastic", seed=9, precision=prec, rng_sharing=sharing)


FIELDS = ("values", "raw", "flagged", "visited_nodes", "path_steps", "path_count")


def _pinned_queries(fs, q):
    """The same queries in page-locked host memory: the H2D copies are then truly
    asynchronous and the host enqueues slab 1 right behind slab 0 (with pageable
    input every copy blocks the host, which hides stream races)."""
    import torch
    buf = torch.empty(q.positions.shape, dtype=torch.float64, pin_memory=True)
    a = buf.numpy()
    a[:] = q.positions
    return fs.QuerySet(a), buf  # (keep buf alive while the QuerySet is used)


@pytest.mark.parametrize("pinned", [False, True], ids=["pageable", "pinned"])
@pytest.mark.parametrize("method,prec,sharing", CASES)
def test_fresh_tree_host_pipeline_equals_device_path(fs, scene, method, prec, sharing, pinned):
    from paper_2506_02219_b200.estimators import evaluate_field_device
    s, q = scene
    keep = None
    if pinned:
        q, keep = _pinned_queries(fs, q)
    kern = fs.KernelSpec("coulomb")
    cfg = _cfg(fs, method, prec, sharing)
    ref = evaluate_field_device(cfg, s, kern, q, fs.build_tree(s, cfg.resolved_branching))
    ref = ref.to_host()
    for rep in range(5):
        fresh = fs.build_tree(s, cfg.resolved_branching)  # never evaluated before
        got = fs.evaluate_field(cfg, s, kern, q, tree=fresh, chunks=8)
        for k in FIELDS:
            np.testing.assert_array_equal(getattr(got, k), getattr(ref, k),
                                          err_msg=f"{method} {prec} {sharing} rep {rep} {k}")


@pytest.mark.parametrize("method,prec,sharing", [CASES[1], CASES[3], CASES[4]])
def test_fresh_tree_two_host_threads(fs, scene, method, prec, sharing):
    """Two host threads make the first call on one fresh tree at the same time
    (ctypes drops the GIL): the lazily packed records are built once, under the
    tree's lock, and both results equal the single-thread evaluation."""
    import torch
    s, q = scene
    kern = fs.KernelSpec("coulomb")
    cfg = _cfg(fs, method, prec, sharing)
    ref = fs.evaluate_field(cfg, s, kern, q, tree=fs.build_tree(s, cfg.resolved_branching))
    ref = {k: np.array(getattr(ref, k)) for k in FIELDS}
    for rep in range(3):
        fresh = fs.build_tree(s, cfg.resolved_branching)
        out, errs = [None, None], []
        gate = threading.Barrier(2)

        def work(i):
            try:
                with torch.cuda.stream(torch.cuda.Stream()):  # a stream per thread
                    gate.wait()
                    r = fs.evaluate_field(cfg, s, kern, q, tree=fresh, chunks=4)
                    out[i] = {k: np.array(getattr(r, k)) for k in FIELDS}
            except Exception as e:  # pragma: no cover - reported below
                errs.append(e)

        th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        for i in range(2):
            for k in FIELDS:
                np.testing.assert_array_equal(out[i][k], ref[k], err_msg=f"thread {i} rep {rep} {k}")


def test_tree_cache_is_per_device_and_thread_safe(fs, scene):
    """evaluate_field without a tree: concurrent first calls on one SourceSet build
    one tree (cache lock) and agree with a prebuilt tree."""
    s0, q = scene
    s = fs.SourceSet(np.array(s0.positions), np.array(s0.masses), np.array(s0.weights))
    kern = fs.KernelSpec("coulomb")
    cfg = fs.EstimatorConfig("stochastic", seed=2, precision="f32")
    qs = fs.QuerySet(q.positions[:200_000])
    ref = np.array(fs.evaluate_field(cfg, s, kern, qs, tree=fs.build_tree(s, 4)).raw)
    out = [None] * 3

    def work(i):
        out[i] = np.array(fs.evaluate_field(cfg, s, kern, qs).raw)

    th = [threading.Thread(target=work, args=(i,)) for i in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in out:
        np.testing.assert_array_equal(r, ref)
