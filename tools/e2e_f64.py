"""e2e of the API-default FP64 stochastic and BH (evaluate_field, pinned C4 queries)
vs the slab count, next to the device-resident call."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev  # noqa: E402
from paper_2506_02219_b200.estimators import evaluate_field_device  # noqa: E402

src, qs, kern = bench.workload()
n = len(qs)
host = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
host.numpy()[:] = qs.positions
qset = fs.QuerySet(host.numpy())
qd = dev.to_device(qs.positions)
CASES = (("sto f64", fs.EstimatorConfig("stochastic", seed=1), 4),
         ("bh f64", fs.EstimatorConfig("barnes_hut", beta=2.0), 2),
         ("bh f32", fs.EstimatorConfig("barnes_hut", beta=2.0, precision="f32"), 2),
         ("bh f32 b6", fs.EstimatorConfig("barnes_hut", beta=6.4, precision="f32"), 2))
for name, cfg, d in CASES[int(os.environ.get("FIRST", "0")):]:
    tree = fs.build_tree(src, d)
    for _ in range(3):
        evaluate_field_device(cfg, src, kern, qd, tree)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        evaluate_field_device(cfg, src, kern, qd, tree)
    torch.cuda.synchronize()
    line = [f"device {(time.perf_counter() - t0) * 100:.3f}"]
    for chunks in (1, 2, 3, 4, 6, 8):
        for _ in range(3):
            fs.evaluate_field(cfg, src, kern, qset, tree=tree, chunks=chunks)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            fs.evaluate_field(cfg, src, kern, qset, tree=tree, chunks=chunks)
        torch.cuda.synchronize()
        line.append(f"{chunks}:{(time.perf_counter() - t0) * 100:.3f}")
    print(name, " ".join(line), "ms", flush=True)
