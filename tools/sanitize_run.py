"""Small end-to-end run of every hot kernel for compute-sanitizer (memcheck /
racecheck / synccheck): tree build d=2/4, FP32 and FP64 stochastic in both stream
modes, the load-balanced and voting BH, brute force, telescoping, moments.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2506_02219_b200 as fs  # noqa: E402
import scenes  # noqa: E402

os.environ.setdefault("FSB_BH_SPLIT_AFTER", "16")  # force BH work items on a small tree
os.environ.setdefault("FSB_BH_MIN_SPLIT", "4")
s = scenes.build_sources(dict(kind="mesh_torus", m=20000, seed=9))
sw = scenes.build_sources(dict(kind="mesh_sphere_winding", m=6000, seed=8, channels=3))
q = fs.QuerySet(np.random.default_rng(1).uniform(-0.8, 0.8, (3000, 3)))
for src, kind in ((s, "coulomb"), (sw, "winding_dipole"), (s, "smooth_exp")):
    kern = fs.KernelSpec(kind)
    t4, t2 = fs.build_tree(src, 4), fs.build_tree(src, 2)
    for prec in ("f32", "f64"):
        for sharing in ("query", "warp"):
            for S in (1, 3):
                fs.evaluate_field(fs.EstimatorConfig("stochastic", samples_per_subdomain=S,
                                                     seed=2, precision=prec,
                                                     rng_sharing=sharing), src, kern, q, tree=t4)
        for vote in (False, True):
            fs.evaluate_field(fs.EstimatorConfig("barnes_hut", beta=2.0, precision=prec,
                                                 bh_warp_vote=vote), src, kern, q, tree=t2)
        fs.evaluate_field(fs.EstimatorConfig("brute_force", precision=prec), src, kern, q)
        fs.evaluate_field(fs.EstimatorConfig("telescoping_exhaustive", precision=prec), src,
                          kern, q, tree=t4)
    # moments (lane groups of 32 at 64 queries, one thread per query at 40,000) and
    # the few-query lane groups of brute force / telescoping (G = 32 at 3,000 queries)
    from paper_2506_02219_b200 import _core
    for nq in (64, 40000):
        qm = np.random.default_rng(3).uniform(-0.8, 0.8, (nq, 3))
        mean, var = np.zeros(nq), np.zeros(nq)
        _core.stochastic_moments_batch(*t4.core_arrays(), fs.estimators.kernel_id(kern),
                                       kern.alpha, kern.distance_floor, qm, 40, 0, np.uint64(3),
                                       mean, var)
print("sanitize run done")
