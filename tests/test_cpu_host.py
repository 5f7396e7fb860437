"""CPU-only checks: the C ABI library and its exported symbols, host-side API
semantics mirrored from the reference's test suite, and the no-CPU-fallback rule."""

import math
import os
import re
import ctypes as C

import numpy as np
import pytest

import paper_2506_02219_b200 as fs
from paper_2506_02219_b200 import _lib, rng, scenes
from paper_2506_02219_b200.kernels import (contribution_rows, kernel_basis, kernel_id,
                                           point_contribution, post_transform)
from golden_data import meta

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fastsum_b200.h")


def _declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fsb_[a-z0-9_]+)\s*\(", text)))


def test_abi_library_loads_and_exports_every_declared_symbol():
    from paper_2506_02219_b200 import _build
    if not os.path.exists(_lib.LIB_PATH):
        _build.build()
    lib = C.CDLL(_lib.LIB_PATH)
    names = _declared_symbols()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), "ctypes signatures must cover the header"
    L = _lib.load(build_if_missing=False)
    assert L.fsb_abi_version() == 2


def test_abi_validates_arguments_without_touching_the_gpu():
    L = _lib.load()
    # null tree handle and bad kernel ids are rejected before any CUDA call
    rc = L.fsb_barnes_hut_batch(None, 0, 200.0, 1e-12, 0, None, 1, None, 2.0, None, None, None)
    assert rc == 1 and b"null tree" in L.fsb_last_error()
    rc = L.fsb_brute_force_batch(7, 200.0, 1e-12, 0, None, None, 1, 1, None, 1, None, None)
    assert rc == 1 and b"kernel id" in L.fsb_last_error()
    rc = L.fsb_brute_force_batch(1, 200.0, 1e-12, 0, None, None, 4, 1, None, 1, None, None)
    assert rc == 1  # winding needs 3 channels
    assert L.fsb_tree_free(None) == 0


def test_host_pipeline_validates_arguments_without_touching_the_gpu():
    """fsb_evaluate_field_host rejects bad arguments (status 1) before any CUDA call."""
    import ctypes as C
    import numpy as np
    L = _lib.load()
    q = np.zeros((4, 3))
    vals = np.zeros(4)
    qp, vp = q.ctypes.data_as(C.c_void_p), vals.ctypes.data_as(C.c_void_p)

    def call(tree=None, values=vp, **kw):
        a = _lib.EvalArgs(method=3, kid=0, alpha=200.0, dfloor=1e-12, precision=1, beta=2.0,
                          n_samples=1, rr_mode=0, seed=1, query_offset=0, smooth=0,
                          query_order=1)
        for k, v in kw.items():
            setattr(a, k, v)
        return L.fsb_evaluate_field_host(tree, C.byref(a), qp, 4, values, None, None, None,
                                         None, None, 2, None)

    assert call(values=None) == 1 and b"null argument" in L.fsb_last_error()
    assert call(method=9) == 1 and b"unknown method" in L.fsb_last_error()
    assert call(kid=5) == 1
    assert call() == 1 and b"null tree" in L.fsb_last_error()          # stochastic needs a tree
    assert call(method=0) == 1 and b"brute force" in L.fsb_last_error()  # needs device sources
    assert call(method=1, beta=0.0) == 1
    assert call(rr_mode=7) == 1
    assert call(rng_group_log2=21) == 1


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    s = fs.SourceSet([[0, 0, 0], [1, 1, 1]], [1.0, 2.0])
    q = fs.QuerySet([[2.0, 0.0, 0.0]])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fs.evaluate_field(fs.EstimatorConfig("brute_force"), s, fs.KernelSpec("coulomb"), q)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fs.build_tree(s)


# ------------------------------------------------------------------ types
def test_types_validation_mirrors_reference():
    p = fs.SourcePoint([0.0, 1.0, 2.0], 2.0, [3.0])
    assert p.mass.shape == (1,) and p.weight == 2.0
    for bad in (([0.0, 1.0], 1.0, [1.0]), ([0, 1, 2], 0.0, [1.0]), ([0, 1, np.inf], 1.0, [1.0])):
        with pytest.raises(ValueError):
            fs.SourcePoint(*bad)
    s = fs.SourceSet([[0, 0, 0], [1, 1, 1]], [2.0, -3.0])
    assert len(s) == 2 and s.channel_count == 1 and s.masses.shape == (2, 1)
    np.testing.assert_array_equal(s.weights, [2.0, 3.0])
    with pytest.raises(AttributeError):
        s.positions = None
    assert not s.positions.flags.writeable
    with pytest.raises(ValueError):
        fs.SourceSet(np.zeros((0, 3)), np.zeros(0))
    with pytest.raises(ValueError):
        fs.SourceSet([[0, 0, 0]], [1.0], weights=[0.0])
    with pytest.raises(ValueError):
        fs.EstimatorConfig("nope")
    with pytest.raises(ValueError):
        fs.EstimatorConfig("barnes_hut", beta=0.0)
    with pytest.raises(ValueError):
        fs.EstimatorConfig("stochastic", samples_per_subdomain=0)
    with pytest.raises(ValueError):
        fs.EstimatorConfig("stochastic", seed=2 ** 64)
    assert fs.EstimatorConfig("barnes_hut").resolved_branching == 2
    assert fs.EstimatorConfig("stochastic").resolved_branching == 4
    with pytest.raises(ValueError):
        fs.KernelSpec("gauss")
    assert fs.KernelSpec("winding_dipole").channel_count == 3
    scale, off, out = fs.normalize_to_unit_cube([[0, 0, 0], [2, 4, 6]])
    assert out.min() >= -1 and out.max() <= 1 and scale == 1 / 3


def test_paper_option_fields_default_to_the_reference():
    """The paper's options are opt-in extensions: defaults reproduce the reference,
    and bad values are rejected like the reference's own config fields."""
    from paper_2506_02219_b200.estimators import _variant
    c = fs.EstimatorConfig("stochastic")
    assert (c.rng_sharing, c.bh_warp_vote, c.path_order) == ("query", False,
                                                             "swap_then_roulette")
    assert _variant(c) == 0
    assert _variant(fs.EstimatorConfig("stochastic", path_order="roulette_then_swap")) == 1
    with pytest.raises(ValueError):
        fs.EstimatorConfig("stochastic", rng_sharing="block")
    with pytest.raises(ValueError):
        fs.EstimatorConfig("stochastic", path_order="random")


# ---------------------------------------------------------------- kernels
def test_kernel_hand_values():
    coul, wind, sm3 = (fs.KernelSpec("coulomb"), fs.KernelSpec("winding_dipole"),
                       fs.KernelSpec("smooth_exp", alpha=3.0))
    assert point_contribution(coul, fs.SourcePoint([2, 0, 0], 1, [1]), [0, 0, 0]) == pytest.approx(-0.5)
    assert point_contribution(coul, fs.SourcePoint([0, 3, 4], 1, [2]), [0, 0, 0]) == pytest.approx(-0.4)
    assert point_contribution(sm3, fs.SourcePoint([1, 0, 0], 1, [1]), [0, 0, 0]) == pytest.approx(math.exp(-3))
    assert point_contribution(wind, fs.SourcePoint([0, 0, 2], 1, [0, 0, 1]), [0, 0, 0]) == \
        pytest.approx(2.0 / (4 * math.pi * 8))
    k = fs.KernelSpec("coulomb", distance_floor=1e-6)
    assert point_contribution(k, fs.SourcePoint([0, 0, 0], 1, [1]), [0, 0, 0]) == pytest.approx(-1e6)
    r = np.random.default_rng(1)
    for kern in (coul, wind, sm3):
        ms = r.normal(size=(5, kern.channel_count))
        for row in range(5):
            p, q = r.uniform(-1, 1, 3), r.uniform(-1, 1, 3)
            got = contribution_rows(kernel_id(kern), kern.alpha, kern.distance_floor, ms, row,
                                    *p, *q)
            assert got == pytest.approx(float(ms[row] @ kernel_basis(kern, p, q).value), rel=1e-14)


def test_post_transform_semantics():
    sm = fs.KernelSpec("smooth_exp", alpha=50.0)
    assert post_transform(sm, 0.0) == (math.inf, True)
    assert post_transform(sm, -1.0) == (math.inf, True)
    v, f = post_transform(sm, math.exp(-5.0))
    assert f is False and v == pytest.approx(0.1)
    assert post_transform(fs.KernelSpec("coulomb"), -3.5) == (-3.5, False)


def test_russian_roulette_and_swap_scalars():
    assert fs.russian_roulette_prob(2.0, 4.0) == 0.5
    assert fs.russian_roulette_prob(0.5, 2.0) == 0.5  # parent ratio clamped to 1
    assert fs.russian_roulette_prob(3.0, 1.0) == 1.0
    assert fs.russian_roulette_prob(3.0, 1.0, "fixed_half") == 0.5
    assert fs.russian_roulette_prob(3.0, 9.0, "disabled") == 1.0
    with pytest.raises(ValueError):
        fs.russian_roulette_prob(-1.0, 1.0)


# -------------------------------------------------------------------- rng
def test_host_rng_matches_reference_goldens():
    for e in meta()["rng"]["keys"]:
        args = [int(a) for a in e["args"]]
        key = rng.stream_key(*args)
        assert key == int(e["key"])
        got = [rng.uniform_draw(key, c) for c in range(8)] + [rng.uniform_draw(key, 2 ** 64 - 1)]
        assert got == e["draws"]
    s = rng.RngStreams(7, 123, 4, 9)
    assert s.index_stream.next_float() == rng.uniform_draw(rng.stream_key(7, 123, 4, 9, 0), 0)
    assert s.roulette_stream.next_float() == rng.uniform_draw(rng.stream_key(7, 123, 4, 9, 1), 0)


# ----------------------------------------------------------------- scenes
def test_scene_generators_match_reference_bytes():
    """make_queries layouts (scene_io.py:188-212): grid z-fastest, slice v-major."""
    g = scenes.make_queries(scenes.GridSpec("grid3d", resolution=(2, 3, 4)))
    assert g.positions.shape == (24, 3)
    assert g.positions[1, 2] > g.positions[0, 2] and g.positions[1, 0] == g.positions[0, 0]
    sl = scenes.make_queries(scenes.GridSpec("slice_plane", resolution=(3, 2), origin=(0, 0, 0.5)))
    assert sl.positions.shape == (6, 3) and np.all(sl.positions[:, 2] == 0.5)
    assert sl.positions[1, 0] > sl.positions[0, 0] and sl.positions[1, 1] == sl.positions[0, 1]
    with pytest.raises(ValueError):
        scenes.GridSpec("slice_plane", u_axis=(1, 1, 0))
    v, f = scenes.icosphere(2, 1.0)
    assert f.shape == (320, 3) and np.allclose(np.linalg.norm(v, axis=1), 1.0)
    src = scenes.sample_mesh_surface(v, f, 1000, seed=3, kernel_kind="winding_dipole")
    assert src.channel_count == 3 and np.allclose(src.weights, src.weights[0])


def test_estimator_api_params_and_clone():
    from sklearn.base import clone
    est = fs.KernelSumEstimator(method="barnes_hut", beta=3.0, seed=4)
    p = est.get_params()
    assert p["beta"] == 3.0 and p["seed"] == 4 and p["method"] == "barnes_hut"
    assert clone(est).get_params() == p


def test_source_set_owns_its_arrays():
    """SourceSet keeps frozen copies of its inputs, so a device tree cached for it
    (evaluate_field without a tree) cannot go stale when the caller later writes
    its own buffer (the reference freezes the caller's arrays in place)."""
    pos = np.random.default_rng(0).uniform(-1, 1, (1000, 3))
    s = fs.SourceSet(pos, np.ones(1000))
    pos[:] = 0.0
    assert not np.all(s.positions == 0.0)
    assert not s.positions.flags.writeable and not s.masses.flags.writeable


def test_pipeline_slab_counts():
    """evaluate_field's default slab count: up to 6 slabs of >= 160 K queries;
    Barnes-Hut fewer (FP32: one -- its work-splitting rounds synchronise with the
    host; FP64: up to three)."""
    import paper_2506_02219_b200 as fs
    from paper_2506_02219_b200.estimators import _pipeline_chunks
    sto = fs.EstimatorConfig("stochastic")
    assert _pipeline_chunks(10, sto) == 1
    assert _pipeline_chunks(10 ** 6, sto) == 6
    assert _pipeline_chunks(10 ** 7, sto) == 6
    assert _pipeline_chunks(10 ** 6, fs.EstimatorConfig("barnes_hut", precision="f32")) == 1
    assert _pipeline_chunks(10 ** 6, fs.EstimatorConfig("barnes_hut")) == 3
    assert _pipeline_chunks(320_000, fs.EstimatorConfig("brute_force")) == 2
    assert _pipeline_chunks(10 ** 6) == 6
