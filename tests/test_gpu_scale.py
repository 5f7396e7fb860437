"""Larger-scale GPU checks: bitwise vs the pinned oracle at 2^16-2^18 sources, and
size-independent properties at the C4 scale (2^22 sources).  Needs a GPU."""

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


KEYS = ("bbox_min", "bbox_max", "diameter", "aggregate_mass", "aggregate_weight",
        "center_of_mass", "child_start", "child_count", "child_index", "begin", "end", "depth",
        "permuted_indices", "points", "masses", "weights")


@pytest.mark.parametrize("d", [2, 4])
def test_tree_2e18_bitwise_vs_oracle(fs, O, d):
    s = scenes.build_sources(dict(kind="mesh_torus", m=2 ** 18, seed=11))
    t = fs.build_tree(s, d)
    ref = O.build_tree(s.positions, s.masses, s.weights, d, 32)
    for k in KEYS:
        np.testing.assert_array_equal(getattr(t, k), ref[k], err_msg=k)


def _structure_ok(t, m):
    n = t.num_nodes
    perm = t.permuted_indices
    assert np.array_equal(np.sort(perm), np.arange(m))
    assert t.begin[0] == 0 and t.end[0] == m
    cc, cs, ci = t.child_count, t.child_start, t.child_index
    assert cs[-1] + cc[-1] == n - 1 and len(ci) == n - 1
    # every non-root node appears exactly once as a child
    assert np.array_equal(np.sort(ci), np.arange(1, n))
    internal = np.nonzero(cc)[0]
    first = ci[cs[internal]]
    assert np.array_equal(first, internal + 1)  # preorder: first child follows its parent
    # children ranges tile the parent: begin(first) = begin(parent), ends chain
    assert np.array_equal(t.begin[first], t.begin[internal])
    # leaves are single points except at the depth cap
    multi = (cc == 0) & (t.end - t.begin > 1)
    assert np.all(t.depth[multi] == t.max_depth)
    # sibling ranges chain: end(child k) == begin(child k+1) inside each parent
    slot_parent = np.repeat(np.arange(n), cc)
    nxt = np.ones(n - 1, dtype=bool)
    nxt[(cs[internal] + cc[internal] - 1)] = False
    idx = np.nonzero(nxt)[0]
    assert np.array_equal(t.end[ci[idx]], t.begin[ci[idx + 1]])
    last = ci[cs[internal] + cc[internal] - 1]
    assert np.array_equal(t.end[last], t.end[internal])
    return slot_parent


def test_c4_scale_tree_properties(fs):
    s = scenes.build_sources(dict(kind="mesh_torus", m=2 ** 22, seed=7))
    for d in (4, 2):
        t = fs.build_tree(s, d)
        m = len(s)
        _structure_ok(t, m)
        # aggregates: root mass = total charge, weights positive, com inside cells
        np.testing.assert_allclose(t.aggregate_mass[0, 0], s.masses.sum(), rtol=1e-12)
        assert np.all(t.aggregate_weight > 0)
        tol = 1e-9
        assert np.all(t.center_of_mass >= t.bbox_min - tol)
        assert np.all(t.center_of_mass <= t.bbox_max + tol)
        # child cell diameter is exactly parent/d up to rounding (octree.py:225)
        cc, cs, ci = t.child_count, t.child_start, t.child_index
        parent = np.repeat(np.arange(t.num_nodes), cc)
        child = ci[np.repeat(cs, cc) + np.concatenate([np.arange(k) for k in cc])]
        np.testing.assert_allclose(t.diameter[child], t.diameter[parent] / d, rtol=1e-12)
        assert np.all(t.depth[child] == t.depth[parent] + 1)


def test_stochastic_and_bh_f64_bitwise_vs_oracle_2e16(fs, O):
    s = scenes.build_sources(dict(kind="mesh_torus", m=2 ** 16, seed=13))
    rng = np.random.default_rng(5)
    q = rng.uniform(-0.6, 0.6, (2048, 3))
    kern = fs.KernelSpec("coulomb")
    for d, method, extra in ((4, "stochastic", dict(seed=9, samples_per_subdomain=2)),
                             (2, "barnes_hut", dict(beta=3.0)),
                             (4, "barnes_hut", dict(beta=1.5, branching_per_dim=4))):
        cfg = fs.EstimatorConfig(method, **extra)
        t = fs.build_tree(s, d)
        r = fs.evaluate_field(cfg, s, kern, fs.QuerySet(q), tree=t)
        ref = O.build_tree(s.positions, s.masses, s.weights, d, 32)
        ca = O.core_arrays(ref)
        out = np.zeros(len(q))
        vis = np.zeros(len(q), dtype=np.int64)
        if method == "barnes_hut":
            O.barnes_hut_batch(*ca, 0, 200.0, 1e-12, q, extra["beta"], 0, out, vis)
        else:
            st = np.zeros(len(q), dtype=np.int64)
            pc = np.zeros(len(q), dtype=np.int64)
            O.stochastic_batch(*ca, 0, 200.0, 1e-12, q, 2, 0, 9, 0, out, vis, st, pc)
            np.testing.assert_array_equal(r.path_steps, st)
        np.testing.assert_array_equal(r.values, out)
        np.testing.assert_array_equal(r.visited_nodes, vis)


def test_statistical_unbiasedness_moments(fs):
    """Acceptance criterion 3 (test_acceptance.py:195-214) on the GPU moments kernel."""
    from paper_2506_02219_b200 import _core
    s = scenes.make_sources(256, seed=31)
    tree = fs.build_tree(s, 4)
    q = scenes.make_query_points(64, seed=32)
    bf = fs.evaluate_field(fs.EstimatorConfig("brute_force"), s, fs.KernelSpec("coulomb"),
                           fs.QuerySet(q))
    n_reps = 100_000
    mean = np.zeros(64)
    var = np.zeros(64)
    _core.stochastic_moments_batch(*tree.core_arrays(), 0, 200.0, 1e-12, q, n_reps, 0,
                                   np.uint64(7), mean, var)
    se = np.sqrt(var * (n_reps / (n_reps - 1)) / n_reps)
    within = np.abs(mean - bf.values) <= 4.0 * se
    assert within.mean() >= 0.95


def test_query_order_and_offset_invariance(fs):
    """Results depend only on (seed, global query index): reordering or slicing the
    query set with the matching query_offset leaves every value unchanged (F8)."""
    from paper_2506_02219_b200.estimators import evaluate_field_device
    s = scenes.build_sources(dict(kind="mesh_torus", m=2 ** 15, seed=17))
    rng = np.random.default_rng(3)
    q = rng.uniform(-0.7, 0.7, (4000, 3))
    t = fs.build_tree(s, 4)
    kern = fs.KernelSpec("coulomb")
    for prec in ("f64", "f32"):
        cfg = fs.EstimatorConfig("stochastic", seed=21, precision=prec)
        full = evaluate_field_device(cfg, s, kern, fs.QuerySet(q), t).to_host().values
        unordered = evaluate_field_device(cfg, s, kern, fs.QuerySet(q), t,
                                          query_order=False).to_host().values
        np.testing.assert_array_equal(full, unordered)
        parts = [evaluate_field_device(cfg, s, kern, fs.QuerySet(q[a:b]), t,
                                       query_offset=a).to_host().values
                 for a, b in ((0, 1500), (1500, 2600), (2600, 4000))]
        np.testing.assert_array_equal(np.concatenate(parts), full)


@pytest.mark.parametrize("method", ["stochastic", "barnes_hut", "brute_force",
                                    "telescoping_exhaustive"])
def test_host_pipeline_slab_invariance(fs, method):
    """evaluate_field (host in / host out, fsb_evaluate_field_host) gives the same
    bytes for any slab count as one device-resident evaluation (F8 + query_offset)."""
    from paper_2506_02219_b200.estimators import evaluate_field_device
    s = scenes.build_sources(dict(kind="mesh_torus", m=2 ** 14, seed=19))
    rng = np.random.default_rng(4)
    q = fs.QuerySet(rng.uniform(-0.7, 0.7, (3001 if method != "telescoping_exhaustive" else 301,
                                            3)))
    for kind in ("coulomb", "smooth_exp"):
        kern = fs.KernelSpec(kind)
        src = s if kind == "coulomb" else fs.SourceSet(s.positions, np.ones((len(s), 1)))
        for prec in ("f64", "f32"):
            extra = dict(seed=5, samples_per_subdomain=2) if method == "stochastic" else {}
            cfg = fs.EstimatorConfig(method, precision=prec, **extra)
            t = None if method == "brute_force" else fs.build_tree(src, cfg.resolved_branching)
            ref = evaluate_field_device(cfg, src, kern, q, t).to_host()
            for chunks in (1, 2, 5):
                r = fs.evaluate_field(cfg, src, kern, q, tree=t, chunks=chunks)
                for k in ("values", "raw", "flagged", "visited_nodes", "path_steps",
                          "path_count"):
                    np.testing.assert_array_equal(getattr(r, k), getattr(ref, k),
                                                  err_msg=f"{method} {kind} {prec} {chunks} {k}")


def test_fast_fp32_estimator_unbiased_over_seeds(fs):
    """Acceptance check 3 on the production kernel: the FP32 stochastic estimator's
    mean over 128 seeds converges to brute force (|mean - truth| <= 4 SE for >= 95 %
    of the queries), and its error shrinks like seeds^-1/2."""
    from paper_2506_02219_b200.estimators import evaluate_field_device
    from paper_2506_02219_b200 import _device as dev
    s = scenes.build_sources(dict(kind="mesh_torus", m=2 ** 16, seed=23))
    rng = np.random.default_rng(6)
    q = rng.uniform(-0.6, 0.6, (2048, 3))
    kern = fs.KernelSpec("coulomb")
    truth = fs.evaluate_field(fs.EstimatorConfig("brute_force"), s, kern, fs.QuerySet(q)).values
    t = fs.build_tree(s, 4)
    qd = dev.to_device(q)
    runs = np.stack([evaluate_field_device(fs.EstimatorConfig("stochastic", seed=k,
                                                              precision="f32"),
                                           s, kern, qd, t).values.cpu().numpy()
                     for k in range(128)])
    mean = runs.mean(axis=0)
    se = runs.std(axis=0, ddof=1) / np.sqrt(len(runs))
    ok = np.abs(mean - truth) <= 4 * se + 1e-6 * np.abs(truth)
    assert ok.mean() >= 0.95, ok.mean()
    e1 = np.median(np.abs(runs[0] - truth))
    e128 = np.median(np.abs(mean - truth))
    assert e128 < e1 / 4  # ~sqrt(128) = 11x in expectation


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_paper_warp_shared_rng_is_unbiased_and_deterministic(fs, prec):
    """rng_sharing="warp" (the paper's GPU recipe): shuffled order,
    32 queries per stream.  Deterministic for a seed, unbiased over seeds, and its
    median error matches the reference-stream estimator's."""
    from paper_2506_02219_b200.estimators import evaluate_field_device
    from paper_2506_02219_b200 import _device as dev
    s = scenes.build_sources(dict(kind="mesh_torus", m=2 ** 15, seed=29))
    rng = np.random.default_rng(8)
    q = rng.uniform(-0.6, 0.6, (4096, 3))
    kern = fs.KernelSpec("coulomb")
    truth = fs.evaluate_field(fs.EstimatorConfig("brute_force"), s, kern, fs.QuerySet(q)).values
    t = fs.build_tree(s, 4)
    qd = dev.to_device(q)

    def run(seed, sharing):
        cfg = fs.EstimatorConfig("stochastic", seed=seed, precision=prec, rng_sharing=sharing)
        return evaluate_field_device(cfg, s, kern, qd, t).values.cpu().numpy()

    np.testing.assert_array_equal(run(3, "warp"), run(3, "warp"))
    runs = np.stack([run(k, "warp") for k in range(64)])
    se = runs.std(axis=0, ddof=1) / np.sqrt(len(runs))
    ok = np.abs(runs.mean(axis=0) - truth) <= 4 * se + 1e-6 * np.abs(truth)
    assert ok.mean() >= 0.95, ok.mean()
    e_warp = np.median([np.median(np.abs(r - truth)) for r in runs[:16]])
    e_ref = np.median([np.median(np.abs(run(k, "query") - truth)) for k in range(16)])
    assert abs(e_warp - e_ref) <= 0.1 * e_ref


def test_tree_reused_for_repeated_calls_on_one_scene(fs, monkeypatch):
    """evaluate_field without a prebuilt tree builds once per (SourceSet, branching)
    and reuses it; a new SourceSet gets its own tree; results are unchanged."""
    from paper_2506_02219_b200 import estimators as E
    calls = []
    real = E.build_tree

    def counting(*a, **k):
        calls.append(1)
        return real(*a, **k)

    monkeypatch.setattr(E, "build_tree", counting)
    s = scenes.build_sources(dict(kind="mesh_torus", m=5000, seed=2))
    q = fs.QuerySet(np.random.default_rng(0).uniform(-0.5, 0.5, (300, 3)))
    kern = fs.KernelSpec("coulomb")
    cfg = fs.EstimatorConfig("stochastic", seed=1)
    a = fs.evaluate_field(cfg, s, kern, q)
    b = fs.evaluate_field(cfg, s, kern, q)
    assert len(calls) == 1
    np.testing.assert_array_equal(a.raw, b.raw)
    fs.evaluate_field(fs.EstimatorConfig("barnes_hut"), s, kern, q)  # d = 2: another tree
    assert len(calls) == 2
    s2 = scenes.build_sources(dict(kind="mesh_torus", m=5000, seed=3))
    fs.evaluate_field(cfg, s2, kern, q)
    assert len(calls) == 3
    ref = fs.evaluate_field(cfg, s, kern, q, tree=fs.build_tree(s, 4))
    np.testing.assert_array_equal(a.raw, ref.raw)


@pytest.mark.parametrize("kind", ["coulomb", "winding_dipole", "smooth_exp"])
def test_fp64_queue_kernel_equals_per_query_kernel(fs, kind, monkeypatch):
    """The FP64 queue kernel (fs_sto64.cu, level-1/2 staged, walks drained by the
    block) and the thread-per-query parity kernel give the same bytes: values and
    all three counters, for every rr mode, S = 1 / 7 / 150 (several drain rounds),
    per-query and warp-shared streams, and a query offset."""
    from paper_2506_02219_b200.estimators import evaluate_field_device
    if kind == "winding_dipole":
        s = scenes.build_sources(dict(kind="mesh_sphere_winding", m=2 ** 15, seed=3))
    else:
        s = scenes.build_sources(dict(kind="mesh_torus", m=2 ** 15, seed=3))
        if kind == "smooth_exp":
            s = fs.SourceSet(s.positions, np.ones((len(s), 1)))
    kern = fs.KernelSpec(kind)
    t = fs.build_tree(s, 4)
    q = fs.QuerySet(np.random.default_rng(9).uniform(-0.8, 0.8, (1500, 3)))
    for S, rr, sharing, off in ((1, "paper_ratio", "query", 0), (7, "fixed_half", "query", 77),
                                (150, "disabled", "query", 0), (1, "paper_ratio", "warp", 0),
                                (3, "paper_ratio", "query", 5)):
        cfg = fs.EstimatorConfig("stochastic", seed=11, samples_per_subdomain=S, rr_mode=rr,
                                 rng_sharing=sharing)
        monkeypatch.delenv("FSB_STO64_OFF", raising=False)
        a = evaluate_field_device(cfg, s, kern, q, t, query_offset=off).to_host()
        monkeypatch.setenv("FSB_STO64_OFF", "1")
        b = evaluate_field_device(cfg, s, kern, q, t, query_offset=off).to_host()
        for k in ("raw", "visited_nodes", "path_steps", "path_count"):
            np.testing.assert_array_equal(getattr(a, k), getattr(b, k),
                                          err_msg=f"{kind} S={S} {rr} {sharing} {k}")
