"""The measurement harness (reference fastsum.bench, bench.py:1-272) mirrored in
paper_2506_02219_b200.bench: host-side semantics on CPU, device statistics and
sweeps on the GPU (checked against the reference's numpy formulas restated here)."""

import numpy as np
import pytest

import paper_2506_02219_b200 as fs
from paper_2506_02219_b200 import bench as B


def _ref_error_stats(est, ref, flags=None):
    """bench.py:66-84 restated: abs errors over unflagged entries, lower median."""
    est = np.asarray(est, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    keep = np.ones(est.shape, bool) if flags is None else ~np.asarray(flags)
    d = np.abs(est[keep] - ref[keep])
    if d.size == 0:
        return (np.nan, np.nan, np.nan, 0)
    return (float(d.mean()), float(np.sort(d)[(d.size - 1) // 2]), float(d.max()), int(d.size))


def test_writers_and_host_helpers(tmp_path):
    st = B.ErrorStats(0.25, 0.125, 1.5, 7)
    recs = [B.SweepRecord("barnes_hut", 2.0, 0.0123, st, 0.5, 12.25, 3, 0.0),
            B.SweepRecord("stochastic", 4.0, 1e-3, st, 0.1, 99.5, 0, 0.375)]
    p = tmp_path / "s.csv"
    B.write_sweep_csv(recs, p)
    lines = p.read_text().splitlines()
    assert lines[0] == ("method,parameter,wall_time_s,mean_abs,median_abs,max_abs,rmse,"
                        "visited_nodes_mean,flagged_count")
    assert lines[1] == "barnes_hut,2,0.0123,0.25,0.125,1.5,0.5,12.25,3"
    labels, acc = B.classify_inside_outside([0.2, 0.7, 0.9], [0.1, 0.4, 0.95])
    assert labels.tolist() == [False, True, True] and acc == pytest.approx(2 / 3)
    with pytest.raises(ValueError):
        B.classify_inside_outside([1.0], [1.0, 2.0])
    with pytest.raises(ValueError):
        B.convergence_slope(recs)  # needs >= 4 points
    four = [B.SweepRecord("stochastic", s, 0.0, st, 1.0 / np.sqrt(s), 1.0, 0) for s in (1, 4, 16, 64)]
    assert B.convergence_slope(four) == pytest.approx(-0.5)
    src = fs.SourceSet(np.zeros((2, 3)) + [[0, 0, 0], [1, 0, 0]], np.ones(2))
    with pytest.raises(ValueError, match="sweeps support"):
        B.run_sweep(src, fs.KernelSpec("coulomb"), "brute_force", [1], fs.QuerySet(np.ones((1, 3))))
    h1 = B.content_hash(src, fs.KernelSpec("coulomb"), fs.QuerySet(np.ones((1, 3))))
    h2 = B.content_hash(src, fs.KernelSpec("smooth_exp"), fs.QuerySet(np.ones((1, 3))))
    assert h1 != h2 and len(h1) == 64


@pytest.mark.gpu
def test_device_error_stats_match_reference_formulas():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(3)
    for n in (1, 2, 7, 1000, 100_001):
        est = rng.normal(size=n)
        ref = rng.normal(size=n)
        flags = rng.random(n) < 0.3
        for fl in (None, flags):
            got = B.error_stats(est, ref, fl)
            want = _ref_error_stats(est, ref, fl)
            if want[3] == 0:
                assert got.count == 0 and np.isnan(got.mean_abs)
                continue
            assert got.count == want[3]
            assert got.median_abs == want[1] and got.max_abs == want[2]  # exact selections
            assert got.mean_abs == pytest.approx(want[0], rel=1e-12)
            keep = np.ones(n, bool) if fl is None else ~fl
            d = est[keep] - ref[keep]
            assert B.rmse(est, ref, fl) == pytest.approx(float(np.sqrt(np.mean(d * d))), rel=1e-12)
    allflag = B.error_stats(np.ones(5), np.zeros(5), np.ones(5, bool))
    assert allflag.count == 0 and np.isnan(allflag.median_abs)
    with pytest.raises(ValueError):
        B.error_stats(np.ones(3), np.ones(4))


@pytest.mark.gpu
def test_sweeps_and_ablation_match_host_statistics(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(9)
    m = 4096
    src = fs.SourceSet(rng.uniform(-0.5, 0.5, (m, 3)), np.full(m, 1.0 / m))
    q = fs.QuerySet(rng.uniform(-1.0, 1.0, (3000, 3)))
    kern = fs.KernelSpec("coulomb")
    oracle = B.oracle_field(src, kern, q)
    bf = fs.evaluate_field(fs.EstimatorConfig("brute_force"), src, kern, q)
    np.testing.assert_array_equal(oracle.values, bf.values)
    assert B.oracle_cache_stats()["misses"] >= 1
    B.oracle_field(src, kern, q)
    assert B.oracle_cache_stats()["hits"] >= 1
    recs = B.run_sweep(src, kern, "barnes_hut", [1.0, 2.0, 4.0], q)
    for r in recs:
        res = fs.evaluate_field(fs.EstimatorConfig("barnes_hut", beta=r.parameter), src, kern, q)
        want = _ref_error_stats(res.values, oracle.values, res.flagged | oracle.flagged)
        assert r.stats.median_abs == want[1] and r.stats.count == want[3]
        assert r.stats.mean_abs == pytest.approx(want[0], rel=1e-12)
        assert r.visited_nodes_mean == pytest.approx(res.visited_nodes.mean())
    assert recs[0].stats.median_abs > recs[-1].stats.median_abs
    srec = B.run_sweep(src, kern, "stochastic", [1, 4, 16, 64], q, seed=5)
    assert B.convergence_slope(srec) < -0.3  # O(S^-1/2) convergence of the RMSE
    abl = B.rr_ablation(src, kern, q, seed=2)
    assert set(abl) == {"paper_ratio", "fixed_half", "disabled"}
    assert abl["disabled"].mean_path_length >= abl["fixed_half"].mean_path_length
    B.write_sweep_json(tmp_path / "s.json", {"scene": "test"}, src, kern, q, recs)
    assert (tmp_path / "s.json").read_text().startswith("{")
