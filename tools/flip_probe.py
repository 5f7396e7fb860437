"""Roulette flips between the FP32 and FP64 stochastic kernels on the same draws:
how many queries flip, and how large their errors are against the brute-force
truth compared with the FP64 kernel's on the same queries."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2506_02219_b200 as fs  # noqa: E402
import scenes  # noqa: E402

CASES = [
    (dict(kind="manydup", m=3000, seed=4, posmass=True), "coulomb"),
    (dict(kind="cluster", m=4000, seed=6, posmass=True), "coulomb"),
    (dict(kind="lattice", m=4096, seed=7), "coulomb"),
    (dict(kind="mesh_sphere_winding", m=6000, seed=8, channels=3), "winding_dipole"),
    (dict(kind="mesh_torus", m=20000, seed=9), "coulomb"),
    (dict(kind="duplicates", m=5000, seed=5, posmass=True), "smooth_exp"),
]
for case, kind in CASES:
    s = scenes.build_sources(case)
    kern = fs.KernelSpec(kind)
    q = fs.QuerySet(np.random.default_rng(11).uniform(-1.2, 1.2, (20000, 3)))
    t = fs.build_tree(s, 4)
    truth = fs.evaluate_field(fs.EstimatorConfig("brute_force"), s, kern, q).raw
    for rr in ("paper_ratio", "fixed_half"):
        for S in (1, 3):
            for sharing in ("query", "warp"):
                cfg = dict(samples_per_subdomain=S, rr_mode=rr, seed=13, rng_sharing=sharing)
                a = fs.evaluate_field(fs.EstimatorConfig("stochastic", precision="f32", **cfg), s, kern, q, tree=t)
                b = fs.evaluate_field(fs.EstimatorConfig("stochastic", precision="f64", **cfg), s, kern, q, tree=t)
                sc = 1.0 + np.abs(truth)
                close = np.abs(a.raw - b.raw) / (1.0 + np.abs(b.raw)) <= 1e-4
                flip = (a.path_steps != b.path_steps) | (a.visited_nodes != b.visited_nodes)
                F = ~close
                ea, eb = np.abs(a.raw - truth) / sc, np.abs(b.raw - truth) / sc
                msg = (f"{case['kind']:>20} {rr:>11} S={S} {sharing:>5}: notclose {F.mean()*100:5.2f}% "
                       f"counters-differ {flip.mean()*100:5.2f}% notclose&counters-same {(F & ~flip).sum():4d}")
                if F.any():
                    msg += (f" | F: med err32 {np.median(ea[F]):.3e} err64 {np.median(eb[F]):.3e} "
                            f"max err32 {ea[F].max():.3e} err64 {eb[F].max():.3e} "
                            f"max |a-b|/sc {np.max(np.abs(a.raw - b.raw)[F] / sc[F]):.3e}")
                msg += f" | all: med err32 {np.median(ea):.3e} err64 {np.median(eb):.3e} max32 {ea.max():.3e} max64 {eb.max():.3e}"
                print(msg, flush=True)
