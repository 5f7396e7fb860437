"""Secondary rows of BASELINE.json's configs on one B200: S=1 stochastic (per-query
streams, and the paper's warp-shared streams) vs the GPU deterministic BH at
matched median error, per config.  C4 is bench.py's
headline.  Writes one JSON line per row to stdout.

    python tools/configs.py [C1 C2s C2t C3 C5]

Ground truth is the GPU brute force (FP32 terms, FP64 accumulation); C5's
error is measured on a 10^6-query subset (the timing uses all 10^7 queries).
"""
import ctypes as C
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev, _lib  # noqa: E402
from paper_2506_02219_b200 import scenes as S  # noqa: E402
from paper_2506_02219_b200.estimators import evaluate_field_device  # noqa: E402
from paper_2506_02219_b200.kernels import kernel_id  # noqa: E402

BETAS = (0.75, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0, 8.0, 10.0, 12.0, 16.0, 24.0)


def scene(name):
    if name == "C1":
        rng = np.random.default_rng(0)
        m = 2 ** 14
        src = fs.SourceSet(rng.uniform(-1, 1, (m, 3)), np.full(m, 1.0 / m))
        q = fs.QuerySet(np.random.default_rng(1).uniform(-1, 1, (4096, 3)))
        return src, q, fs.KernelSpec("coulomb"), "rel", "2^14 uniform masses, 4096 random queries"
    if name in ("C2s", "C2t"):
        if name == "C2s":
            v, f = S.icosphere(5, 0.5)
            desc = "icosphere(5, 0.5)"
        else:
            v, f = S.torus(0.5, 0.15)
            v = S.rotate_x(v, 0.7)
            desc = "torus(0.5, 0.15) tilted 0.7 rad"
        src = S.sample_mesh_surface(v, f, 2 ** 20, seed=2, kernel_kind="winding_dipole")
        q = S.make_queries(S.GridSpec("slice_plane", resolution=(512, 512), origin=(0, 0, 0.03)))
        return (src, q, fs.KernelSpec("winding_dipole"), "abs",
                f"winding number, 2^20 samples of {desc}, 512^2 slice z=0.03")
    if name == "C3":
        v, f = S.icosphere(5, 0.5)
        src = S.sample_mesh_surface(v, f, 2 ** 20, seed=2, kernel_kind="smooth_exp",
                                    point_mass=1.0)
        q = S.make_queries(S.GridSpec("grid3d", resolution=(256, 256, 256)))
        return (src, q, fs.KernelSpec("smooth_exp"), "abs_unflagged",
                "smooth distance (alpha=200), 2^20 samples of icosphere(5, 0.5), 256^3 grid")
    if name == "C5":
        v, f = S.torus(0.25, 0.06)
        v = S.rotate_x(v, 0.7) + np.array([0.1, 0.05, -0.1])
        src = S.sample_mesh_surface(v, f, 2 ** 24, seed=7, kernel_kind="coulomb")
        q = fs.QuerySet(np.random.default_rng(5).uniform(-1, 1, (10 ** 7, 3)))
        return (src, q, fs.KernelSpec("coulomb"), "rel",
                "coulomb, 2^24 tilted-torus samples, 10^7 random queries (1 GPU)")
    raise ValueError(name)


CLOCKS = []  # (label, clocks summary) of every timed region


def timed(fn, reps=3, label="", trials=3):
    """Best of `trials` means over `reps` calls (CUDA events), after one warm-up call."""
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    with bench.Clocks(torch.cuda.current_device()) as clk:
        clk.active = True
        for _ in range(trials):
            a.record()
            for _ in range(reps):
                r = fn()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            best = ms if best is None else min(best, ms)
        clk.active = False
    CLOCKS.append((label, clk.summary()))
    return best, r


def error(kind, est, truth, flagged_t=None, flagged_e=None):
    if kind == "rel":
        return float(np.median(np.abs(est - truth) / np.abs(truth)))
    if kind == "abs":
        return float(np.median(np.abs(est - truth)))
    ok = ~(flagged_t | flagged_e)
    return float(np.median(np.abs(est[ok] - truth[ok])))


def run(name):
    src, qs, kern, ekind, desc = scene(name)
    L = _lib.lib()
    n = len(qs)
    q = dev.to_device(qs.positions)
    sub = slice(0, n) if n <= 2_000_000 else slice(0, n, n // 1_000_000)
    qsub = dev.to_device(qs.positions[sub])
    # ground truth (values after the post-transform, like FieldResult.values)
    pts, ms = dev.to_device(src.positions), dev.to_device(src.masses)
    raw = dev.empty(qsub.shape[0], torch.float64)
    t0 = time.perf_counter()
    _lib.check(L.fsb_brute_force_f32acc64(kernel_id(kern), kern.alpha,
                                           kern.distance_floor, C.c_void_p(dev.ptr(pts)),
                                           C.c_void_p(dev.ptr(ms)), len(src), src.channel_count,
                                           C.c_void_p(dev.ptr(qsub)), qsub.shape[0],
                                           C.c_void_p(dev.ptr(raw)), C.c_void_p(dev.stream_ptr())))
    torch.cuda.synchronize()
    truth_s = time.perf_counter() - t0
    traw = raw.cpu().numpy()
    if kern.kind == "smooth_exp":
        tflag = traw <= 0
        with np.errstate(divide="ignore"):
            tval = np.where(tflag, np.inf, -np.log(np.where(tflag, 1.0, traw)) / kern.alpha)
    else:
        tflag, tval = np.zeros(len(traw), bool), traw

    def err_of(r):
        v = r.values.cpu().numpy()[sub]
        f = r.flagged.cpu().numpy().astype(bool)[sub]
        return error(ekind, v, tval, tflag, f)

    t4, t2 = fs.build_tree(src, 4), fs.build_tree(src, 2)
    cfg = fs.EstimatorConfig("stochastic", seed=1, precision="f32")
    s1_ms, r = timed(lambda: evaluate_field_device(cfg, src, kern, q, t4), label="s1")
    s1_err = err_of(r)
    # the paper's GPU recipe: warp-shared streams over a shuffled order
    cfg_w = fs.EstimatorConfig("stochastic", seed=1, precision="f32", rng_sharing="warp")
    w_ms, rw = timed(lambda: evaluate_field_device(cfg_w, src, kern, q, t4), label="s1_warp")
    w_err = err_of(rw)
    sweep = []
    for beta in BETAS:
        cfgb = fs.EstimatorConfig("barnes_hut", beta=beta, precision="f32")
        ms_b, rb = timed(lambda: evaluate_field_device(cfgb, src, kern, q, t2), reps=2,
                         label=f"bh{beta}")
        e = err_of(rb)
        sweep.append({"beta": beta, "ms": ms_b, "err": e,
                      "visited_mean": float(rb.visited.double().mean().item())})
        if e < 0.5 * min(s1_err, w_err) or ms_b > 20000:
            break
    matched = bench.loglog_interp([(p["err"], p["ms"]) for p in sweep], s1_err)
    matched_w = bench.loglog_interp([(p["err"], p["ms"]) for p in sweep], w_err)
    row = {"config": name, "workload": desc, "queries": n, "sources": len(src),
           "error_metric": {"rel": "median relative error", "abs": "median absolute error",
                            "abs_unflagged": "median absolute error of values, unflagged"}[ekind],
           "truth": f"GPU brute force f32/f64-acc ({truth_s:.1f} s"
                    + (", 10^6-query subset)" if sub.step else ")"),
           "s1_ms": s1_ms, "s1_queries_per_s": n / (s1_ms * 1e-3), "s1_err": s1_err,
           "bh_sweep": sweep, "matched_bh_ms": matched,
           "speedup_at_matched_error": (matched / s1_ms) if matched else None,
           "warp_streams": {"s1_ms": w_ms, "s1_queries_per_s": n / (w_ms * 1e-3),
                            "s1_err": w_err, "matched_bh_ms": matched_w,
                            "speedup_at_matched_error": (matched_w / w_ms) if matched_w else None}}
    mins = [c.get("sm_mhz_min") for _, c in CLOCKS if c.get("sm_mhz_min")]
    reasons = sorted({x for _, c in CLOCKS for x in c.get("reasons", [])})
    row["clocks"] = {"sm_mhz_min": min(mins) if mins else None, "reasons": reasons}
    CLOCKS.clear()
    if kern.kind == "smooth_exp":
        row["flagged_fraction"] = float(r.flagged.double().mean().item())
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    for name in (sys.argv[1:] or ["C1", "C2s", "C2t", "C3", "C5"]):
        run(name)
