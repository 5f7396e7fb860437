"""The reference's end-to-end acceptance gate (tests/test_acceptance.py, 10 criteria),
restated on the GPU path through the same public API.  Criterion 2 (exact
expectation by enumeration) is covered by the draw-for-draw parity with the oracle
(test_gpu_parity.py) and criterion 3 by test_gpu_scale.py; criterion 10 (worker
counts) becomes slab/block/GPU-count determinism here.  Needs a GPU."""

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
def sphere_scene(fs):
    from paper_2506_02219_b200 import scenes as S
    verts, faces = S.icosphere(subdivisions=4, radius=0.25)
    src = S.sample_mesh_surface(verts, faces, 2 ** 15, seed=1, kernel_kind="coulomb")
    return src, S.make_queries(S.GridSpec("grid3d", resolution=(50, 50, 50)))


@pytest.fixture(scope="module")
def sphere_sweep(fs, sphere_scene):
    from paper_2506_02219_b200 import bench as B
    src, q = sphere_scene
    return B.run_sweep(src, fs.KernelSpec("coulomb"), "stochastic", [1, 4, 16, 64, 256], q,
                       seed=3)


def test_criterion_01_telescoping_identity(fs):
    """test_acceptance.py:92-109: telescoping equals brute force to 1e-9 on 20 scenes."""
    worst = 0.0
    for i in range(20):
        m = (16, 256, 4096)[i % 3]
        d = (2, 4)[i % 2]
        s = scenes.make_sources(m, seed=i)
        q = fs.QuerySet(scenes.make_query_points(100, seed=1000 + i))
        bf = fs.evaluate_field(fs.EstimatorConfig("brute_force"), s, fs.KernelSpec("coulomb"), q)
        tel = fs.evaluate_field(fs.EstimatorConfig("telescoping_exhaustive", branching_per_dim=d),
                                s, fs.KernelSpec("coulomb"), q)
        worst = max(worst, float((np.abs(tel.values - bf.values) / (1 + np.abs(bf.values))).max()))
    assert worst <= 1e-9, worst


def test_criterion_04_barnes_hut_limits(fs):
    """test_acceptance.py:221-242: beta -> inf is brute force (1e-10); a beta below the
    root's far-field ratio returns exactly the root term."""
    kern = fs.KernelSpec("coulomb")
    worst = 0.0
    for i in range(10):
        s = scenes.make_sources((64, 256, 1024)[i % 3], seed=400 + i)
        q = fs.QuerySet(scenes.make_query_points(20, seed=500 + i))
        bf = fs.evaluate_field(fs.EstimatorConfig("brute_force"), s, kern, q)
        bh = fs.evaluate_field(fs.EstimatorConfig("barnes_hut", beta=1e9), s, kern, q)
        worst = max(worst, float((np.abs(bh.values - bf.values) / (1 + np.abs(bf.values))).max()))
    assert worst <= 1e-10
    s = scenes.make_sources(256, seed=499)
    tree = fs.build_tree(s, branching_per_dim=2)
    far_q = np.array([40.0, -25.0, 60.0])
    beta = fs.far_field_ratio(tree.root, far_q) * 0.5
    assert fs.barnes_hut(tree, s, kern, far_q, beta) == fs.node_contribution(kern, tree.root, far_q)


def test_criterion_05_monte_carlo_rate(fs, sphere_sweep):
    """test_acceptance.py:249-254: RMSE slope over S in {1..256} in [-0.65, -0.35]."""
    from paper_2506_02219_b200 import bench as B
    slope = B.convergence_slope(sphere_sweep)
    assert -0.65 <= slope <= -0.35, slope


@pytest.mark.parametrize("sharing", ["query", "warp"])
def test_criterion_06_error_ordering(fs, sphere_scene, sphere_sweep, sharing):
    """test_acceptance.py:261-271: S=1 beats BH beta=2 in mean error and by >= 5x in
    median error (the reference streams; and the paper's shared streams in FP32)."""
    from paper_2506_02219_b200 import bench as B
    src, q = sphere_scene
    kern = fs.KernelSpec("coulomb")
    if sharing == "query":
        sto = next(r for r in sphere_sweep if r.parameter == 1.0).stats
    else:
        truth = B.oracle_field(src, kern, q)
        r = fs.evaluate_field(fs.EstimatorConfig("stochastic", seed=3, precision="f32",
                                                 rng_sharing="warp"), src, kern, q)
        sto = B.error_stats(r.values, truth.values)
    bh = B.run_sweep(src, kern, "barnes_hut", [2.0], q)[0].stats
    assert sto.mean_abs < bh.mean_abs
    assert bh.median_abs / sto.median_abs >= 5.0


def test_criterion_07_roulette_ablation(fs):
    """test_acceptance.py:278-289: paper_ratio roulette at most halves node visits vs
    disabled, at no more than 3x the error."""
    from paper_2506_02219_b200 import bench as B, scenes as S
    verts, faces = S.torus(0.6, 0.08)
    src = S.sample_mesh_surface(verts, faces, 2 ** 15, seed=1, kernel_kind="coulomb")
    q = S.make_queries(S.GridSpec("grid3d", resolution=(50, 50, 50)))
    out = B.rr_ablation(src, fs.KernelSpec("coulomb"), q, seed=9)
    node_ratio = out["paper_ratio"].visited_nodes_mean / out["disabled"].visited_nodes_mean
    err_ratio = out["paper_ratio"].stats.mean_abs / out["disabled"].stats.mean_abs
    assert node_ratio <= 0.5 and err_ratio <= 3.0, (node_ratio, err_ratio)


@pytest.mark.parametrize("prec,sharing", [("f64", "query"), ("f32", "query"), ("f32", "warp")])
def test_criterion_08_winding_classification(fs, prec, sharing):
    """test_acceptance.py:296-314: inside/outside accuracy >= 0.99 at S=16 and >= 0.95
    at S=1 against brute-force labels (2^17 oriented samples, 50^3 grid)."""
    from paper_2506_02219_b200 import bench as B, scenes as S
    verts, faces = S.icosphere(subdivisions=4, radius=0.7)
    src = S.sample_mesh_surface(verts, faces, 2 ** 17, seed=2, kernel_kind="winding_dipole")
    q = S.make_queries(S.GridSpec("grid3d", resolution=(50, 50, 50)))
    kern = fs.KernelSpec("winding_dipole")
    labels = B.oracle_field(src, kern, q).values > 0.5
    acc = {}
    for s_count in (16, 1):
        r = fs.evaluate_field(fs.EstimatorConfig("stochastic", samples_per_subdomain=s_count,
                                                 seed=5, precision=prec, rng_sharing=sharing),
                              src, kern, q)
        acc[s_count] = float(np.mean((r.values > 0.5) == labels))
    assert acc[16] >= 0.99 and acc[1] >= 0.95, acc


def test_criterion_09_smooth_distance(fs):
    """test_acceptance.py:321-350: a single source gives the exact distance through
    every method; telescoping matches brute force through the post-transform."""
    kern = fs.KernelSpec("smooth_exp", alpha=50.0)
    src = fs.SourceSet([[0.25, -0.5, 0.75]], [1.0])
    q = fs.QuerySet(scenes.make_query_points(20, seed=900))
    true_d = np.linalg.norm(q.positions - src.positions[0], axis=1)
    for method in ("brute_force", "stochastic", "barnes_hut", "telescoping_exhaustive"):
        r = fs.evaluate_field(fs.EstimatorConfig(method), src, kern, q)
        assert np.all(np.abs(r.values - true_d) <= 1e-10), method
        assert r.flagged_count == 0
    s = scenes.make_sources(500, seed=901)
    s = fs.SourceSet(s.positions, np.abs(s.masses) + 0.1)
    bf = fs.evaluate_field(fs.EstimatorConfig("brute_force"), s, kern, q)
    tel = fs.evaluate_field(fs.EstimatorConfig("telescoping_exhaustive"), s, kern, q)
    assert np.max(np.abs(tel.values - bf.values) / (1 + np.abs(bf.values))) <= 1e-9
    hand = np.array([fs.post_transform(kern, r)[0] for r in tel.raw])
    np.testing.assert_array_equal(hand, tel.values)


@pytest.mark.parametrize("prec,sharing", [("f64", "query"), ("f32", "query"), ("f32", "warp")])
def test_criterion_10_determinism(fs, prec, sharing):
    """test_acceptance.py:380-404 (byte-identical across worker counts), on the GPU:
    the same call repeated, split into 1/3/8 host-pipeline slabs, or into query
    slabs with query_offset gives byte-identical values."""
    s = scenes.make_sources(4096, seed=1010)
    kern = fs.KernelSpec("coulomb")
    q = scenes.make_query_points(3 * (1 << 16) + 77, seed=7)
    t = fs.build_tree(s, 4)
    cfg = fs.EstimatorConfig("stochastic", samples_per_subdomain=2, seed=7, precision=prec,
                             rng_sharing=sharing)
    ref = fs.evaluate_field(cfg, s, kern, fs.QuerySet(q), tree=t, chunks=1)
    for chunks in (1, 3, 8):
        r = fs.evaluate_field(cfg, s, kern, fs.QuerySet(q), tree=t, chunks=chunks)
        assert r.values.tobytes() == ref.values.tobytes()
    # query slabs (the multi-GPU partition; window-aligned for shared streams)
    from paper_2506_02219_b200.sharding import SHUFFLE_WINDOW, slab
    align = SHUFFLE_WINDOW if sharing == "warp" else 1
    parts = []
    for rank in range(3):
        a, b = slab(len(q), rank, 3, align)
        parts.append(fs.evaluate_field(cfg, s, kern, fs.QuerySet(q[a:b]), tree=t,
                                       query_offset=a).values)
    assert np.concatenate(parts).tobytes() == ref.values.tobytes()
