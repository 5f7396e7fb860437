"""e2e (pinned C4 queries, evaluate_field) vs the host pipeline's slab count."""
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
n = len(qs)
host = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
host.numpy()[:] = qs.positions
qset = fs.QuerySet(host.numpy())
for sharing in ("warp", "query"):
    cfg = fs.EstimatorConfig("stochastic", seed=1, precision="f32", rng_sharing=sharing)
    for rep in range(2):
        line = []
        for chunks in (2, 3, 4, 5, 6, 8, 12):
            for _ in range(3):
                fs.evaluate_field(cfg, src, kern, qset, tree=tree, chunks=chunks)
            ts = []
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(10):
                    fs.evaluate_field(cfg, src, kern, qset, tree=tree, chunks=chunks)
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t0) / 10 * 1e3)
            line.append(f"{chunks}:{np.median(ts):.3f}")
        print(sharing, " ".join(line), flush=True)
