"""e2e (host in / host out) timing of evaluate_field on the C4 workload vs slab count."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200.estimators import evaluate_field_device  # noqa: E402

src, qs, kern = bench.workload()
tree = fs.build_tree(src, 4)
host = torch.empty((len(qs), 3), dtype=torch.float64, pin_memory=True)
host.numpy()[:] = qs.positions
qset = fs.QuerySet.__new__(fs.QuerySet)
object.__setattr__(qset, "positions", host.numpy())
cfg = fs.EstimatorConfig("stochastic", seed=1, precision="f32")
ref = evaluate_field_device(cfg, src, kern, qset, tree).to_host()
for ch in [int(x) for x in os.environ.get("CHUNKS", "1,2,3,4,6,8").split(",")]:
    for _ in range(3):
        r = fs.evaluate_field(cfg, src, kern, qset, tree=tree, chunks=ch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        r = fs.evaluate_field(cfg, src, kern, qset, tree=tree, chunks=ch)
    dt = (time.perf_counter() - t0) / 10
    same = np.array_equal(r.values, ref.values) and np.array_equal(r.visited_nodes, ref.visited_nodes)
    print(f"chunks={ch}: {dt*1e3:.3f} ms/step, identical to one launch: {same}", flush=True)
