"""GPU parity against the reference goldens and the pinned oracle (needs a B200).

FP64 ("parity") mode must reproduce the reference bit for bit for coulomb and
winding (tree topology and aggregates always bitwise); smooth_exp within a few
ulp (exp/log).  All calls go through the package API / the C ABI.
"""

import numpy as np
import pytest

from golden_data import TREE_KEYS, arrays, case_id, digest, meta, parse_sto
import scenes

pytestmark = pytest.mark.gpu

KINDS = {"coulomb": 0, "winding_dipole": 1, "smooth_exp": 2}


@pytest.fixture(scope="module")
def fs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_02219_b200 as fs
    return fs


def _assert_close(got, ref, kernel, what):
    if kernel == "smooth_exp":
        np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-300, err_msg=what)
    else:
        np.testing.assert_array_equal(got, ref, err_msg=what)


@pytest.mark.parametrize("case", meta()["small_trees"], ids=case_id)
def test_gpu_tree_small_bitwise(fs, case):
    A = arrays()
    pre = case["prefix"]
    s = fs.SourceSet(A[pre + "in_positions"], A[pre + "in_masses"], A[pre + "in_weights"])
    t = fs.build_tree(s, case["d"], case["max_depth"])
    for k in TREE_KEYS:
        got = getattr(t, k)
        np.testing.assert_array_equal(got, A[pre + k], err_msg=k)
        assert got.dtype == A[pre + k].dtype, k
    if case["kind"] != "coincident":  # the reference validator flags a zero-side root leaf too
        assert fs.validate_tree(t, s) == []


@pytest.mark.parametrize("case", meta()["large_trees"], ids=case_id)
def test_gpu_tree_large_digest(fs, case):
    s = scenes.build_sources(case)
    t = fs.build_tree(s, case["d"], case["max_depth"])
    for k in TREE_KEYS:
        assert digest(getattr(t, k)) == case["arrays"][k], k


@pytest.mark.parametrize("entry", meta()["cores"], ids=lambda e: e["prefix"])
def test_gpu_cores_match_reference(fs, entry):
    from paper_2506_02219_b200 import _core
    A = arrays()
    pre = entry["prefix"]
    pos, ms, w, q = (A[pre + k] for k in ("positions", "masses", "weights", "queries"))
    kid, alpha = KINDS[entry["kernel"]], entry.get("alpha", 200.0)
    n = q.shape[0]
    out = np.zeros(n)
    _core.brute_force_batch(kid, alpha, 1e-12, pos, ms, q, out)
    _assert_close(out, A[pre + "brute"], entry["kernel"], "brute")
    md = entry.get("max_depth", 32)
    src = fs.SourceSet(pos, ms, w)
    for d in (2, 4):
        tree = fs.build_tree(src, d, md)
        ca = tree.core_arrays()
        for run in entry["runs"]:
            if f"_d{d}" not in run:
                continue
            out = np.zeros(n)
            vis = np.zeros(n, dtype=np.int64)
            if run.startswith("bh_"):
                beta = float(run.split("_b")[-1])
                _core.barnes_hut_batch(*ca, kid, alpha, 1e-12, q, beta, 0, out, vis)
                _assert_close(out, A[pre + run], entry["kernel"], run)
                np.testing.assert_array_equal(vis, A[pre + run + "_visited"])
            elif run.startswith("tel_"):
                _core.telescoping_batch(*ca, kid, alpha, 1e-12, q, out, vis)
                _assert_close(out, A[pre + run], entry["kernel"], run)
                np.testing.assert_array_equal(vis, A[pre + run + "_visited"])
            elif run.startswith("sto_"):
                S, rr, seed, off = parse_sto(run)
                st = np.zeros(n, dtype=np.int64)
                pc = np.zeros(n, dtype=np.int64)
                _core.stochastic_batch(*ca, kid, alpha, 1e-12, q, S, rr, np.uint64(seed), off, out,
                                       vis, st, pc)
                _assert_close(out, A[pre + run], entry["kernel"], run)
                np.testing.assert_array_equal(vis, A[pre + run + "_visited"])
                np.testing.assert_array_equal(st, A[pre + run + "_steps"])
                np.testing.assert_array_equal(pc, A[pre + run + "_count"])
            elif run.startswith("mom_"):
                var = np.zeros(n)
                _core.stochastic_moments_batch(*ca, kid, alpha, 1e-12, q, 50, 0, np.uint64(7),
                                               out, var)
                _assert_close(out, A[pre + run + "_mean"], entry["kernel"], run)
                if entry["kernel"] == "smooth_exp":
                    # var = E[t^2] - mean^2 cancels: ulp-level exp differences are amplified
                    scale = float(np.max(A[pre + run + "_mean"] ** 2))
                    np.testing.assert_allclose(var, A[pre + run + "_var"], rtol=1e-6,
                                               atol=1e-12 * scale)
                else:
                    _assert_close(var, A[pre + run + "_var"], entry["kernel"], run + " var")


@pytest.mark.parametrize("entry", meta()["cores"][:3], ids=lambda e: e["prefix"])
def test_gpu_evaluate_field_device_tree_matches_reference(fs, entry):
    """evaluate_field on the GPU-built tree (no core-array round trip)."""
    A = arrays()
    pre = entry["prefix"]
    pos, ms, w, q = (A[pre + k] for k in ("positions", "masses", "weights", "queries"))
    src = fs.SourceSet(pos, ms, w)
    kern = fs.KernelSpec(entry["kernel"], alpha=entry.get("alpha", 200.0))
    qs = fs.QuerySet(q)
    r = fs.evaluate_field(fs.EstimatorConfig("barnes_hut", beta=2.0), src, kern, qs)
    _assert_close(r.raw, A[pre + "bh_d2_b2"], entry["kernel"], "bh")
    np.testing.assert_array_equal(r.visited_nodes, A[pre + "bh_d2_b2_visited"])
    r = fs.evaluate_field(fs.EstimatorConfig("stochastic", samples_per_subdomain=3, seed=11),
                          src, kern, qs)
    _assert_close(r.raw, A[pre + "sto_d4_S3_rr0_seed11_off0"], entry["kernel"], "sto")
    np.testing.assert_array_equal(r.visited_nodes, A[pre + "sto_d4_S3_rr0_seed11_off0_visited"])


@pytest.mark.gpu
def test_fp64_branch_free_div_sqrt_bitwise_equal_intrinsics():
    """The FP64 queue kernel's branch-free division / square root (fs_common.cuh
    ddiv_fast / dsqrt_fast) must equal __ddiv_rn / __dsqrt_rn bit for bit whenever
    they claim the fast path (else the kernel recomputes with the intrinsic)."""
    import ctypes as C
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_02219_b200 import _lib
    counts = (C.c_ulonglong * 4)()
    for seed in (1, 2, 3):
        _lib.check(_lib.lib().fsb_selftest_fp64(1 << 24, seed, counts))
        div_ok, div_bad, sqrt_ok, sqrt_bad = list(counts)
        assert div_bad == 0 and sqrt_bad == 0, list(counts)
        assert div_ok > (1 << 23) and sqrt_ok > (1 << 23)  # the fast path is the common case


def test_fp64_bh_acceptance_shortcut_equals_reference_test():
    """k_bh<F64> decides _ffr(q, node) >= beta (_core.py:44-52, 117) from d2 against
    (beta dm)^2 (1 +- 2^-46) and runs the reference's sqrt / division only inside
    that band: the decision must equal the reference's on queries placed within a
    few ulps of the acceptance sphere, within 1e-9 of it, and anywhere, including
    sub-floor diameters and betas from 2^-600 to 2^600."""
    import ctypes as C
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_02219_b200 import _lib
    counts = (C.c_ulonglong * 2)()
    for seed in (1, 2, 3):
        _lib.check(_lib.lib().fsb_selftest_bh_far(1 << 24, seed, counts))
        assert counts[0] == 1 << 24 and counts[1] == 0, list(counts)

