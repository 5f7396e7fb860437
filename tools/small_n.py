"""Device-path time of the API-default FP64 kernels (and FP32) at small query
counts: C1 (2^14 uniform sources, 4096 queries) and C4 subsets."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev  # noqa: E402
from paper_2506_02219_b200.estimators import evaluate_field_device  # noqa: E402

rng = np.random.default_rng(0)
c1 = fs.SourceSet(rng.uniform(-1, 1, (2 ** 14, 3)), np.full((2 ** 14, 1), 1.0 / 2 ** 14))
q1 = dev.to_device(np.random.default_rng(1).uniform(-1, 1, (4096, 3)))
src4, qs4, _ = bench.workload()
kern = fs.KernelSpec("coulomb")
cases = [("C1", c1, q1)] + [(f"C4[{n}]", src4, dev.to_device(qs4.positions[:n].copy())) for n in (1000, 16384)]
for name, src, q in cases:
    t4, t2 = fs.build_tree(src, 4), fs.build_tree(src, 2)
    cases_k = (("sto f64", fs.EstimatorConfig("stochastic", seed=1), t4),
               ("sto f32", fs.EstimatorConfig("stochastic", seed=1, precision="f32"), t4),
               ("sto f32 warp", fs.EstimatorConfig("stochastic", seed=1, precision="f32",
                                                   rng_sharing="warp"), t4),
               ("bh f64", fs.EstimatorConfig("barnes_hut", beta=2.0), t2))
    only = os.environ.get("ONLY")
    for label, cfg, t in cases_k:
        if only and label != only:
            continue
        for _ in range(3):
            evaluate_field_device(cfg, src, kern, q, t)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            evaluate_field_device(cfg, src, kern, q, t)
        b.record()
        torch.cuda.synchronize()
        print(f"{os.path.basename(os.environ.get('FSB_LIB', 'default')):>10} {name:>10} {label}: "
              f"{a.elapsed_time(b) / 10:.3f} ms", flush=True)
