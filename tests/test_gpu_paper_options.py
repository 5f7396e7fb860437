"""The paper's GPU options (not in the reference), checked against the
oracle's restatement of the paper's algorithm: warp-voting Barnes-Hut
and warp-shared RNG streams.  FP64 bitwise vs the oracle; FP32
vs FP64 to FP32 rounding.  Needs a GPU."""

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


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    return oracle


CASES = [
    (dict(kind="mesh_torus", m=20000, seed=9), "coulomb"),
    (dict(kind="manydup", m=3000, seed=4, posmass=True), "coulomb"),
    (dict(kind="mesh_sphere_winding", m=6000, seed=8, channels=3), "winding_dipole"),
    (dict(kind="duplicates", m=5000, seed=5, posmass=True), "smooth_exp"),
]
KID = {"coulomb": 0, "winding_dipole": 1, "smooth_exp": 2}


def _same(a, b, kind):
    """Bitwise for coulomb/winding; smooth_exp to 1e-10 relative, 1e-13 of the field's
    scale absolute (device exp vs glibc exp, amplified by cancelling swaps)."""
    if kind == "smooth_exp":
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-13 * np.abs(b).max())
    else:
        np.testing.assert_array_equal(a, b)


def _morton(fs, qd, n):
    import torch
    from paper_2506_02219_b200 import _device as dev, _lib
    p = dev.empty(n, torch.int32)
    _lib.check(_lib.lib().fsb_query_order(C.c_void_p(dev.ptr(qd)), n, C.c_void_p(dev.ptr(p)),
                                          C.c_void_p(dev.stream_ptr())))
    return p.cpu().numpy()


@pytest.mark.parametrize("case,kind", CASES, ids=lambda c: c if isinstance(c, str) else c["kind"])
def test_vote_bh_f64_bitwise_vs_oracle(fs, O, case, kind):
    from paper_2506_02219_b200.estimators import evaluate_field_device
    from paper_2506_02219_b200 import _device as dev
    s = scenes.build_sources(case)
    kern = fs.KernelSpec(kind)
    q = np.random.default_rng(3).uniform(-1.1, 1.1, (1000, 3))
    n = len(q)
    qd = dev.to_device(q)
    t = fs.build_tree(s, 2)
    ca = t.core_arrays()
    for beta in (1.0, 2.0, 6.0):
        cfg = fs.EstimatorConfig("barnes_hut", beta=beta, bh_warp_vote=True)
        for morton in (False, True):
            r = evaluate_field_device(cfg, s, kern, qd, t, query_order=morton)
            order = _morton(fs, qd, n) if morton else None
            out, vis = np.zeros(n), np.zeros(n, dtype=np.int64)
            O.barnes_hut_vote_batch(*ca, KID[kind], kern.alpha, kern.distance_floor, q, order,
                                    beta, out, vis)
            _same(r.raw.cpu().numpy(), out, kind)
            np.testing.assert_array_equal(r.visited.cpu().numpy(), vis)


@pytest.mark.parametrize("split", ["1", "0"], ids=["split", "warp"])
@pytest.mark.parametrize("case,kind", CASES, ids=lambda c: c if isinstance(c, str) else c["kind"])
def test_vote_bh_f32_matches_f64_vote(fs, case, kind, split, monkeypatch):
    """FP32 voting BH (load-balanced split kernel, or the warp-coherent one) walks
    the FP64 voting BH's node sets (up to acceptance tests at the FP32 boundary)
    and agrees to 1e-5 * (1 + |ref|) where the sets agree."""
    from paper_2506_02219_b200.estimators import evaluate_field_device
    from paper_2506_02219_b200 import _device as dev
    monkeypatch.setenv("FSB_BH_SPLIT", split)
    monkeypatch.setenv("FSB_BH_SPLIT_AFTER", "16")  # force items on small trees
    monkeypatch.setenv("FSB_BH_MIN_SPLIT", "4")
    s = scenes.build_sources(case)
    kern = fs.KernelSpec(kind)
    qd = dev.to_device(np.random.default_rng(5).uniform(-1.1, 1.1, (3000, 3)))
    t = fs.build_tree(s, 2)
    for beta in (1.0, 4.0):
        a = evaluate_field_device(fs.EstimatorConfig("barnes_hut", beta=beta, precision="f32",
                                                     bh_warp_vote=True), s, kern, qd, t)
        b = evaluate_field_device(fs.EstimatorConfig("barnes_hut", beta=beta, precision="f64",
                                                     bh_warp_vote=True), s, kern, qd, t)
        va, vb = a.visited.cpu().numpy(), b.visited.cpu().numpy()
        same = va == vb
        assert same.mean() >= 0.9, same.mean()
        ra, rb = a.raw.cpu().numpy(), b.raw.cpu().numpy()
        fin = np.isfinite(rb) & same
        assert (np.abs(ra[fin] - rb[fin]) / (1 + np.abs(rb[fin]))).max() <= 1e-5


def test_vote_bh_is_more_accurate_and_host_pipeline_matches(fs):
    """Voting opens a superset of each query's nodes: error at a given beta is no
    worse than per-query BH's (median), and evaluate_field (host pipeline, one
    slab) returns the device path's values bit for bit."""
    from paper_2506_02219_b200.estimators import evaluate_field_device
    from paper_2506_02219_b200 import _device as dev
    s = scenes.build_sources(dict(kind="mesh_torus", m=30000, seed=3))
    kern = fs.KernelSpec("coulomb")
    q = np.random.default_rng(6).uniform(-0.6, 0.6, (20000, 3))
    t = fs.build_tree(s, 2)
    truth = fs.evaluate_field(fs.EstimatorConfig("brute_force"), s, kern, fs.QuerySet(q)).values
    for prec in ("f32", "f64"):
        cfg_v = fs.EstimatorConfig("barnes_hut", beta=3.0, precision=prec, bh_warp_vote=True)
        cfg_p = fs.EstimatorConfig("barnes_hut", beta=3.0, precision=prec)
        rv = fs.evaluate_field(cfg_v, s, kern, fs.QuerySet(q), tree=t, chunks=4)
        rp = fs.evaluate_field(cfg_p, s, kern, fs.QuerySet(q), tree=t)
        assert (rv.visited_nodes >= rp.visited_nodes).mean() > 0.99
        ev = np.median(np.abs(rv.values - truth) / np.abs(truth))
        ep = np.median(np.abs(rp.values - truth) / np.abs(truth))
        assert ev <= ep
        rd = evaluate_field_device(cfg_v, s, kern, dev.to_device(q), t).to_host()
        np.testing.assert_array_equal(rv.raw, rd.raw)
        np.testing.assert_array_equal(rv.visited_nodes, rd.visited_nodes)


@pytest.mark.parametrize("rr", ["paper_ratio", "fixed_half", "disabled"])
@pytest.mark.parametrize("case,kind", CASES, ids=lambda c: c if isinstance(c, str) else c["kind"])
def test_warp_shared_streams_f64_bitwise_vs_oracle(fs, O, case, kind, rr):
    """rng_sharing="warp" in FP64 (k_stochastic with group keys) against the oracle
    with keys[order[t]] = (t + query_offset) >> 5: values and counters bitwise."""
    import torch
    from paper_2506_02219_b200.estimators import evaluate_field_device
    from paper_2506_02219_b200 import _device as dev, _lib
    s = scenes.build_sources(case)
    kern = fs.KernelSpec(kind)
    q = np.random.default_rng(7).uniform(-1.1, 1.1, (700, 3))
    n = len(q)
    qd = dev.to_device(q)
    t = fs.build_tree(s, 4)
    ca = t.core_arrays()
    codes = {"paper_ratio": 0, "fixed_half": 1, "disabled": 2}
    for S, seed, off in ((1, 11, 0), (3, 12, 64), (2, 2 ** 64 - 1, 7)):
        cfg = fs.EstimatorConfig("stochastic", samples_per_subdomain=S, rr_mode=rr, seed=seed,
                                 rng_sharing="warp")
        r = evaluate_field_device(cfg, s, kern, qd, t, query_offset=off)
        p = dev.empty(n, torch.int32)
        _lib.check(_lib.lib().fsb_shuffle_order(n, seed, off, C.c_void_p(dev.ptr(p)),
                                                C.c_void_p(dev.stream_ptr())))
        order = p.cpu().numpy().astype(np.int64)
        keys = np.zeros(n, dtype=np.uint64)
        keys[order] = ((np.arange(n) + off) >> 5).astype(np.uint64)
        res = [np.zeros(n)] + [np.zeros(n, dtype=np.int64) for _ in range(3)]
        O.stochastic_ex_batch(*ca, KID[kind], kern.alpha, kern.distance_floor, q, S, codes[rr],
                              seed, 0, *res, keys=keys)
        _same(r.raw.cpu().numpy(), res[0], kind)
        np.testing.assert_array_equal(r.visited.cpu().numpy(), res[1])
        np.testing.assert_array_equal(r.path_steps.cpu().numpy(), res[2])
        np.testing.assert_array_equal(r.path_count.cpu().numpy(), res[3])


@pytest.mark.parametrize("rr", ["paper_ratio", "fixed_half"])
@pytest.mark.parametrize("case,kind", CASES, ids=lambda c: c if isinstance(c, str) else c["kind"])
def test_alg2_walk_f64_bitwise_vs_oracle(fs, O, case, kind, rr):
    """path_order="roulette_then_swap" (the paper's Alg. 2) in FP64 against the oracle:
    values and counters bitwise, alone and combined with warp-shared streams; the FP32
    generic kernel tracks it to FP32 rounding."""
    import torch
    from paper_2506_02219_b200.estimators import evaluate_field_device
    from paper_2506_02219_b200 import _device as dev, _lib
    s = scenes.build_sources(case)
    kern = fs.KernelSpec(kind)
    q = np.random.default_rng(9).uniform(-1.1, 1.1, (600, 3))
    n = len(q)
    qd = dev.to_device(q)
    t = fs.build_tree(s, 4)
    ca = t.core_arrays()
    codes = {"paper_ratio": 0, "fixed_half": 1, "disabled": 2}
    for S, seed, off, sharing in ((1, 5, 0, "query"), (3, 6, 40, "query"), (2, 7, 64, "warp")):
        res = {}
        for prec in ("f64", "f32"):
            cfg = fs.EstimatorConfig("stochastic", samples_per_subdomain=S, rr_mode=rr, seed=seed,
                                     rng_sharing=sharing, path_order="roulette_then_swap",
                                     precision=prec)
            res[prec] = evaluate_field_device(cfg, s, kern, qd, t, query_offset=off)
        keys = None
        if sharing == "warp":
            p = dev.empty(n, torch.int32)
            _lib.check(_lib.lib().fsb_shuffle_order(n, seed, off, C.c_void_p(dev.ptr(p)),
                                                    C.c_void_p(dev.stream_ptr())))
            order = p.cpu().numpy().astype(np.int64)
            keys = np.zeros(n, dtype=np.uint64)
            keys[order] = ((np.arange(n) + off) >> 5).astype(np.uint64)
        ref = [np.zeros(n)] + [np.zeros(n, dtype=np.int64) for _ in range(3)]
        O.stochastic_ex_batch(*ca, KID[kind], kern.alpha, kern.distance_floor, q, S, codes[rr],
                              seed, off, *ref, keys=keys, variant=1)
        r = res["f64"]
        _same(r.raw.cpu().numpy(), ref[0], kind)
        np.testing.assert_array_equal(r.visited.cpu().numpy(), ref[1])
        np.testing.assert_array_equal(r.path_steps.cpu().numpy(), ref[2])
        np.testing.assert_array_equal(r.path_count.cpu().numpy(), ref[3])
        a = res["f32"].raw.cpu().numpy()
        fin = np.isfinite(ref[0])
        close = np.abs(a[fin] - ref[0][fin]) / (1 + np.abs(ref[0][fin])) <= 1e-4
        assert close.mean() >= 0.97, close.mean()


@pytest.mark.parametrize("n", [1, 2, 31, 33, 65537])
def test_warp_shared_small_and_ragged_query_counts(fs, O, n):
    """k_sto_warp with partial chunks and a partial last shuffle window: FP32 values
    track the FP64 shared-key path, counters agree, every query is written once."""
    from paper_2506_02219_b200.estimators import evaluate_field_device
    from paper_2506_02219_b200 import _device as dev
    s = scenes.build_sources(dict(kind="mesh_torus", m=20000, seed=9))
    kern = fs.KernelSpec("coulomb")
    q = np.random.default_rng(n).uniform(-0.7, 0.7, (n, 3))
    qd = dev.to_device(q)
    t = fs.build_tree(s, 4)
    r = {}
    for prec in ("f32", "f64"):
        cfg = fs.EstimatorConfig("stochastic", seed=5, precision=prec, rng_sharing="warp")
        r[prec] = evaluate_field_device(cfg, s, kern, qd, t, query_offset=32 * n)
    a, b = r["f32"].raw.cpu().numpy(), r["f64"].raw.cpu().numpy()
    assert np.isfinite(a).all() and (a != 0).all()
    close = np.abs(a - b) / (1 + np.abs(b)) <= 1e-4
    assert close.mean() >= 0.97
    same = r["f32"].path_steps.cpu().numpy() == r["f64"].path_steps.cpu().numpy()
    assert same.mean() >= 0.97
    ref = [np.zeros(n)] + [np.zeros(n, dtype=np.int64) for _ in range(3)]
    O.stochastic_ex_batch(*t.core_arrays(), 0, 200.0, 1e-12, q, 1, 0, 5, 0, *ref,
                          keys=O.shared_keys(n, 5, 32 * n))
    np.testing.assert_array_equal(b, ref[0])


def test_ex_entry_validates_flags(fs):
    """fsb_stochastic_batch_ex: unknown flags, or FSB_FLAG_SHUFFLED with an explicit
    order, are argument errors (status 1, ValueError in Python)."""
    import ctypes as C
    import torch
    from paper_2506_02219_b200 import _device as dev, _lib
    s = scenes.build_sources(dict(kind="mesh_torus", m=5000, seed=1))
    t = fs.build_tree(s, 4)
    h = C.c_void_p(t._device_tree().handle)
    q = dev.to_device(np.zeros((64, 3)))
    out = dev.empty(64, torch.float32)
    order = dev.empty(64, torch.int32)
    L = _lib.lib()
    sp = C.c_void_p(dev.stream_ptr())

    def call(order_ptr, flags):
        return L.fsb_stochastic_batch_ex(h, 0, 200.0, 1e-12, 1, C.c_void_p(dev.ptr(q)), 64,
                                         order_ptr, 1, 0, 1, 0, 5, flags,
                                         C.c_void_p(dev.ptr(out)), None, None, None, sp)

    assert call(None, 4) == 1 and b"flags" in L.fsb_last_error()
    assert call(C.c_void_p(dev.ptr(order)), 2) == 1 and b"order = NULL" in L.fsb_last_error()
    assert call(None, 2) == 0 and call(None, 3) == 0


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_alg2_host_pipeline_equals_device_path(fs, prec):
    """path_order="roulette_then_swap" through evaluate_field (pipelined slabs, with and
    without shared streams) gives the device path's values and counters bit for bit."""
    from paper_2506_02219_b200.estimators import evaluate_field_device
    from paper_2506_02219_b200 import _device as dev
    s = scenes.build_sources(dict(kind="mesh_torus", m=20000, seed=5))
    kern = fs.KernelSpec("coulomb")
    q = np.random.default_rng(6).uniform(-0.6, 0.6, (2 * (1 << 16) + 300, 3))
    t = fs.build_tree(s, 4)
    for sharing in ("query", "warp"):
        cfg = fs.EstimatorConfig("stochastic", seed=8, precision=prec, rng_sharing=sharing,
                                 path_order="roulette_then_swap")
        ref = evaluate_field_device(cfg, s, kern, dev.to_device(q), t).to_host()
        r = fs.evaluate_field(cfg, s, kern, fs.QuerySet(q), tree=t, chunks=3)
        np.testing.assert_array_equal(r.raw, ref.raw)
        np.testing.assert_array_equal(r.path_steps, ref.path_steps)
