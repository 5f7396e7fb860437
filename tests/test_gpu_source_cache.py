"""Device copies of a SourceSet's arrays are cached while it lives
(octree.device_sources): repeated builds / brute-force evaluations of one scene
reuse them, a new SourceSet replaces them, and results are unchanged.  Needs a GPU."""

import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_02219_b200 as fs
    return fs


def test_device_sources_cache(fs):
    from paper_2506_02219_b200.octree import device_sources, _SRC_CACHE
    rng = np.random.default_rng(5)
    s = fs.SourceSet(rng.uniform(-1, 1, (5000, 3)), rng.normal(size=5000))
    a = device_sources(s)
    b = device_sources(s)
    assert all(x is y for x, y in zip(a, b))
    np.testing.assert_array_equal(a[0].cpu().numpy(), s.positions)
    np.testing.assert_array_equal(a[1].cpu().numpy().reshape(s.masses.shape), s.masses)
    np.testing.assert_array_equal(a[2].cpu().numpy(), s.weights)
    t1, t2 = fs.build_tree(s, 4), fs.build_tree(s, 4)  # the second build reads the cache
    for k in ("child_start", "begin", "end", "points", "aggregate_mass", "center_of_mass"):
        np.testing.assert_array_equal(getattr(t1, k), getattr(t2, k), err_msg=k)
    s2 = fs.SourceSet(rng.uniform(-1, 1, (3000, 3)), rng.normal(size=3000))
    c = device_sources(s2)
    assert c[0].shape[0] == 3000 and _SRC_CACHE["src"]() is s2  # only the latest is kept
    q = fs.QuerySet(rng.uniform(-1, 1, (200, 3)))
    cfg = fs.EstimatorConfig("brute_force")
    r1 = fs.evaluate_field(cfg, s2, fs.KernelSpec("coulomb"), q)
    r2 = fs.evaluate_field(cfg, s2, fs.KernelSpec("coulomb"), q)
    np.testing.assert_array_equal(r1.values, r2.values)
    del s2, c
    gc.collect()
    assert "src" not in _SRC_CACHE  # freed with its SourceSet
