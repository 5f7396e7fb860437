"""e2e probe: the bench's pinned and pageable evaluate_field steps (C4, warp-shared
streams) for the library in FSB_LIB, three trials of 20 steps each."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402

src, qs, kern = bench.workload()
tree = fs.build_tree(src, 4)
cfg = fs.EstimatorConfig("stochastic", seed=1, precision="f32", rng_sharing="warp")
n = len(qs)
host = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
host.numpy()[:] = qs.positions
tag = os.path.basename(os.environ.get("FSB_LIB", "default"))
if os.environ.get("PROF"):  # a CUPTI session first, as bench.py's launch count
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]):
        fs.evaluate_field(cfg, src, kern, fs.QuerySet(host.numpy()), tree=tree)
        torch.cuda.synchronize()
    tag += "+prof"
for name, qset in (("pinned", fs.QuerySet(host.numpy())), ("pageable", fs.QuerySet(np.array(qs.positions)))):
    res = []
    for trial in range(3):
        for _ in range(3):
            r = fs.evaluate_field(cfg, src, kern, qset, tree=tree)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            r = fs.evaluate_field(cfg, src, kern, qset, tree=tree)
        torch.cuda.synchronize()
        res.append((time.perf_counter() - t0) / 20 * 1e3)
    print(f"{tag:>12} {name:>8}: " + " ".join(f"{x:.3f}" for x in res) + " ms/step", flush=True)
