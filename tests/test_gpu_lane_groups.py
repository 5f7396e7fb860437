"""The few-query launch shapes of the FP64 brute force, telescoping and moments
kernels (G = 8 or 32 lanes per query below 75,776 queries, one thread per query
above) give every query the same bits: a query's result depends only on the query
(_core.py:80-98, 132-156, 270-336 are per-query loops), never on the batch size
that picked the launch shape.
"""

import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu

N_BIG = 80_000  # one thread per query (>= 148 x 16 x 32 queries)
N_MID = 20_000  # 8 lanes per query
N_SMALL = 3_000  # 32 lanes per query


@pytest.fixture(scope="module")
def fs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_02219_b200 as fs
    return fs


@pytest.fixture(scope="module")
def scene(fs):
    s = scenes.build_sources(dict(kind="mesh_torus", m=4096, seed=21))
    q = np.random.default_rng(22).uniform(-0.7, 0.7, (N_BIG, 3))
    return s, q, fs.build_tree(s, 4)


@pytest.mark.parametrize("method", ["brute_force", "telescoping_exhaustive"])
def test_launch_shapes_agree(fs, scene, method):
    s, q, tree = scene
    kern = fs.KernelSpec("coulomb")
    cfg = fs.EstimatorConfig(method)
    big = fs.evaluate_field(cfg, s, kern, fs.QuerySet(q), tree=tree)
    for n in (N_MID, N_SMALL):
        part = fs.evaluate_field(cfg, s, kern, fs.QuerySet(q[:n]), tree=tree)
        np.testing.assert_array_equal(part.raw, big.raw[:n], err_msg=f"{method} n={n}")
        np.testing.assert_array_equal(part.visited_nodes, big.visited_nodes[:n])


def test_moments_launch_shapes_agree(fs, scene):
    from paper_2506_02219_b200 import _core
    s, q, tree = scene
    reps = 40

    def moments(qq):
        mean, var = np.zeros(len(qq)), np.zeros(len(qq))
        _core.stochastic_moments_batch(*tree.core_arrays(), 0, 200.0, 1e-12, qq, reps, 0,
                                       np.uint64(9), mean, var)
        return mean, var

    mean_b, var_b = moments(q)
    for n in (N_MID, N_SMALL):
        mean, var = moments(q[:n])
        np.testing.assert_array_equal(mean, mean_b[:n], err_msg=f"n={n}")
        np.testing.assert_array_equal(var, var_b[:n], err_msg=f"n={n}")
