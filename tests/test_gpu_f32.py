"""precision="f32" path vs the reference's precision="f32" / "f64" runs (needs a GPU).

North-star bar: brute force and deterministic BH within 1e-5 * (1 + |ref|)
of the reference (FP32 inputs, written in each assertion); the stochastic
estimator draws the same index streams, so almost every query reproduces the
reference's f32 estimate to FP32 rounding, and its median error vs brute force
stays within 5 % of the reference's.
"""

import os

import numpy as np
import pytest

from golden_data import arrays, meta
import scenes

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def fs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_02219_b200 as fs
    return fs


def _setup(fs, entry):
    s = scenes.build_sources(entry["src"])
    kern = fs.KernelSpec(entry["kernel"], alpha=entry.get("alpha", 200.0))
    q = fs.QuerySet(arrays()[entry["prefix"] + "queries"])
    return s, kern, q


def _rel(a, b):
    return np.abs(a - b) / (1.0 + np.abs(b))


@pytest.mark.parametrize("entry", meta()["f32"], ids=lambda e: e["kernel"])
def test_f32_brute_force_within_1e5(fs, entry):
    A = arrays()
    s, kern, q = _setup(fs, entry)
    r = fs.evaluate_field(fs.EstimatorConfig("brute_force", precision="f32"), s, kern, q)
    ref64 = A[entry["prefix"] + "brute_force__f64_raw"]
    ref32 = A[entry["prefix"] + "brute_force__f32_raw"]
    assert _rel(r.raw, ref64).max() <= TOL
    assert _rel(r.raw, ref32).max() <= TOL
    assert r.raw.dtype == np.float64 and np.all(r.visited_nodes == len(s))


@pytest.mark.parametrize("beta", [2.0, 4.0])
@pytest.mark.parametrize("entry", meta()["f32"], ids=lambda e: e["kernel"])
def test_f32_barnes_hut_matches_reference(fs, entry, beta):
    A = arrays()
    s, kern, q = _setup(fs, entry)
    r = fs.evaluate_field(fs.EstimatorConfig("barnes_hut", beta=beta, precision="f32"), s, kern, q)
    tag = entry["prefix"] + f"barnes_hut_beta{beta}"
    ref32 = A[tag + "_f32_raw"]
    ref64 = A[tag + "_f64_raw"]
    same_set = r.visited_nodes == A[tag + "_f32_visited"]
    # acceptance tests near the threshold may flip in FP32 (the reference's own f32
    # mode differs from its f64 mode the same way); everything else agrees to 1e-5
    assert same_set.mean() >= 0.98
    assert _rel(r.raw, ref32)[same_set].max() <= TOL
    assert _rel(r.raw, ref64)[same_set].max() <= TOL


@pytest.mark.parametrize("fast", [True, False], ids=["fast", "generic"])
@pytest.mark.parametrize("entry", meta()["f32"], ids=lambda e: e["kernel"])
def test_f32_stochastic_tracks_reference(fs, entry, fast, monkeypatch):
    if not fast:
        monkeypatch.setenv("FSB_DISABLE_FAST", "1")
    A = arrays()
    s, kern, q = _setup(fs, entry)
    truth = A[entry["prefix"] + "brute_force__f64_raw"]
    for extra, tag in ((dict(seed=3), "stochastic_seed3"),
                       (dict(seed=3, samples_per_subdomain=4),
                        "stochastic_seed3_samples_per_subdomain4")):
        r = fs.evaluate_field(fs.EstimatorConfig("stochastic", precision="f32", **extra), s,
                              kern, q)
        ref = A[entry["prefix"] + tag + "_f64_raw"]
        close = _rel(r.raw, ref) <= TOL
        assert close.mean() >= 0.95, close.mean()
        e_ours = np.median(np.abs(r.raw - truth))
        e_ref = np.median(np.abs(ref - truth))
        assert abs(e_ours - e_ref) <= 0.05 * e_ref + 1e-12


def test_f32_outputs_match_reference_dtype_contract(fs):
    entry = meta()["f32"][0]
    s, kern, q = _setup(fs, entry)
    r = fs.evaluate_field(fs.EstimatorConfig("stochastic", precision="f32"), s, kern, q)
    # raw is stored in FP32 and reported as float64 (estimators.py:273, 320)
    assert r.raw.dtype == np.float64
    assert np.array_equal(r.raw, r.raw.astype(np.float32).astype(np.float64))
    assert r.path_count.min() >= 1 and r.flagged.dtype == bool
