"""Pin the C oracle (oracle/fastsum_oracle.c) against the reference's goldens.

CPU only.  The oracle is the checker for every GPU parity test, so it must
reproduce the imported reference bit for bit first (coulomb/winding; the
smooth kernel within a few ulp because exp() may differ in the last bit).
"""

import numpy as np
import pytest

from golden_data import TREE_KEYS, arrays, case_id, digest, meta, parse_sto
from oracle import oracle as O
import scenes

KINDS = {"coulomb": 0, "winding_dipole": 1, "smooth_exp": 2}


@pytest.mark.parametrize("case", meta()["small_trees"], ids=case_id)
def test_oracle_small_trees_bitwise(case):
    A = arrays()
    pre = case["prefix"]
    t = O.build_tree(A[pre + "in_positions"], A[pre + "in_masses"], A[pre + "in_weights"],
                     case["d"], case["max_depth"])
    for k in TREE_KEYS:
        np.testing.assert_array_equal(t[k], A[pre + k], err_msg=k)
        assert t[k].dtype == A[pre + k].dtype, k


@pytest.mark.parametrize("case", meta()["large_trees"], ids=case_id)
def test_oracle_large_trees_digest(case):
    s = scenes.build_sources(case)
    for k in ("positions", "masses", "weights"):
        assert digest(getattr(s, k)) == case["inputs"][k], f"input regenerator drift: {k}"
    t = O.build_tree(s.positions, s.masses, s.weights, case["d"], case["max_depth"])
    for k in TREE_KEYS:
        assert digest(t[k]) == case["arrays"][k], k


def test_oracle_rng_keys_and_draws():
    for e in meta()["rng"]["keys"]:
        args = [int(a) for a in e["args"]]
        key = O.stream_key(*args)
        assert key == int(e["key"])
        got = [O.uniform_draw(key, c) for c in range(8)] + [O.uniform_draw(key, 2 ** 64 - 1)]
        assert got == e["draws"]


def test_np_pairwise_sum_replica():
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(1, 600))
        a = rng.normal(size=n) * np.exp(5 * rng.normal(size=n))
        assert O.np_sum(a) == float(a.sum())


def _core_inputs(entry):
    A = arrays()
    pre = entry["prefix"]
    return (A[pre + "positions"], A[pre + "masses"], A[pre + "weights"], A[pre + "queries"],
            KINDS[entry["kernel"]], entry.get("alpha", 200.0))


def _assert_close(got, ref, kernel, what):
    if kernel == "smooth_exp":
        np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-300, err_msg=what)
    else:
        np.testing.assert_array_equal(got, ref, err_msg=what)


@pytest.mark.parametrize("entry", meta()["cores"], ids=lambda e: e["prefix"])
def test_oracle_cores_match_reference(entry):
    A = arrays()
    pre = entry["prefix"]
    pos, ms, w, q, kid, alpha = _core_inputs(entry)
    n = q.shape[0]
    out = np.zeros(n)
    O.brute_force_batch(kid, alpha, 1e-12, pos, ms, q, out)
    _assert_close(out, A[pre + "brute"], entry["kernel"], "brute")
    md = entry.get("max_depth", 32)
    for d in (2, 4):
        t = O.build_tree(pos, ms, w, d, md)
        ca = O.core_arrays(t)
        for run in entry["runs"]:
            if not run.endswith(f"_d{d}") and f"_d{d}_" not in run:
                continue
            out = np.zeros(n)
            vis = np.zeros(n, dtype=np.int64)
            if run.startswith("bh_"):
                beta = float(run.split("_b")[-1])
                O.barnes_hut_batch(*ca, kid, alpha, 1e-12, q, beta, (md + 2) * d ** 3 + 8, out, vis)
                _assert_close(out, A[pre + run], entry["kernel"], run)
                np.testing.assert_array_equal(vis, A[pre + run + "_visited"])
            elif run.startswith("tel_"):
                O.telescoping_batch(*ca, kid, alpha, 1e-12, q, out, vis)
                _assert_close(out, A[pre + run], entry["kernel"], run)
                np.testing.assert_array_equal(vis, A[pre + run + "_visited"])
            elif run.startswith("sto_"):
                S, rr, seed, off = parse_sto(run)
                st = np.zeros(n, dtype=np.int64)
                pc = np.zeros(n, dtype=np.int64)
                O.stochastic_batch(*ca, kid, alpha, 1e-12, q, S, rr, seed, off, out, vis, st, pc)
                _assert_close(out, A[pre + run], entry["kernel"], run)
                np.testing.assert_array_equal(vis, A[pre + run + "_visited"])
                np.testing.assert_array_equal(st, A[pre + run + "_steps"])
                np.testing.assert_array_equal(pc, A[pre + run + "_count"])
            elif run.startswith("mom_"):
                var = np.zeros(n)
                O.stochastic_moments_batch(*ca, kid, alpha, 1e-12, q, 50, 0, 7, out, var)
                _assert_close(out, A[pre + run + "_mean"], entry["kernel"], run)
                _assert_close(var, A[pre + run + "_var"], entry["kernel"], run + " var")


def _small_tree(seed=3, m=3000, d=2):
    s = scenes.build_sources(dict(kind="mesh_torus", m=m, seed=seed))
    t = O.build_tree(s.positions, s.masses, s.weights, d, 32)
    return s, O.core_arrays(t)


def test_oracle_vote_bh_properties():
    """The warp-voting BH restatement: at beta -> inf it equals the
    reference's BH bitwise (every node opened down to the leaves either way); at
    finite beta each query's node set contains its own BH set (visited >=) and the
    group shares one count."""
    s, ca = _small_tree()
    q = np.random.default_rng(2).uniform(-0.6, 0.6, (200, 3))
    n = len(q)
    for beta in (1e9, 2.0):
        a, va = np.zeros(n), np.zeros(n, dtype=np.int64)
        b, vb = np.zeros(n), np.zeros(n, dtype=np.int64)
        O.barnes_hut_batch(*ca, 0, 200.0, 1e-12, q, beta, 0, a, va)
        O.barnes_hut_vote_batch(*ca, 0, 200.0, 1e-12, q, None, beta, b, vb)
        if beta > 1e8:
            np.testing.assert_array_equal(a, b)
            np.testing.assert_array_equal(va, vb)
        else:
            assert (vb >= va).all() and (vb > va).any()
            for g in range(0, n, 32):
                assert len(set(vb[g:g + 32])) == 1
    # the group order matters only through the grouping
    order = np.random.default_rng(5).permutation(n).astype(np.int32)
    c, vc = np.zeros(n), np.zeros(n, dtype=np.int64)
    O.barnes_hut_vote_batch(*ca, 0, 200.0, 1e-12, q, order, 2.0, c, vc)
    for g in range(0, n, 32):
        assert len(set(vc[order[g:g + 32]])) == 1


def test_oracle_keyed_stochastic_reduces_to_reference():
    """keys[i] = i + offset reproduces stochastic_batch exactly; a shared key gives
    every query of the group the same sampled paths (same path_count)."""
    s, ca = _small_tree(d=4)
    q = np.random.default_rng(4).uniform(-0.6, 0.6, (64, 3))
    n = len(q)
    ref = [np.zeros(n)] + [np.zeros(n, dtype=np.int64) for _ in range(3)]
    O.stochastic_batch(*ca, 0, 200.0, 1e-12, q, 2, 0, 9, 100, *ref)
    got = [np.zeros(n)] + [np.zeros(n, dtype=np.int64) for _ in range(3)]
    O.stochastic_ex_batch(*ca, 0, 200.0, 1e-12, q, 2, 0, 9, 0, *got,
                          keys=np.arange(n, dtype=np.uint64) + 100)
    for x, y in zip(ref, got):
        np.testing.assert_array_equal(x, y)


def test_oracle_alg2_walk_is_unbiased():
    """The paper's Alg. 2 (roulette before each swap): the mean over many keys
    converges to brute force (an unbiased estimator, like the reference's walk)."""
    s, ca = _small_tree(d=4, m=2000)
    q = np.random.default_rng(8).uniform(-0.7, 0.7, (8, 3))
    n = len(q)
    truth = np.zeros(n)
    O.brute_force_batch(0, 200.0, 1e-12, s.positions, s.masses, q, truth)
    reps = 4000
    runs = np.zeros((reps, n))
    for r in range(reps):
        out = [np.zeros(n)] + [np.zeros(n, dtype=np.int64) for _ in range(3)]
        O.stochastic_ex_batch(*ca, 0, 200.0, 1e-12, q, 1, 0, 17, r * n, *out, variant=1)
        runs[r] = out[0]
    se = runs.std(axis=0, ddof=1) / np.sqrt(reps)
    assert (np.abs(runs.mean(axis=0) - truth) <= 4 * se + 1e-9 * np.abs(truth)).all()
    # it differs from the reference walk draw for draw
    ref = [np.zeros(n)] + [np.zeros(n, dtype=np.int64) for _ in range(3)]
    O.stochastic_batch(*ca, 0, 200.0, 1e-12, q, 1, 0, 17, 0, *ref)
    assert not np.array_equal(ref[0], runs[0])
