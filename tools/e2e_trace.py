"""Per-slab timeline of one evaluate_field call (FSB_TRACE=1): C4, warp-shared
streams, pinned queries; prints the library's slab lines and the wall time."""
import os
import sys
import time

os.environ["FSB_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402

src, qs, kern = bench.workload()
tree = fs.build_tree(src, 4)
sharing = os.environ.get("SHARING", "warp")
cfg = fs.EstimatorConfig("stochastic", seed=1, precision="f32", rng_sharing=sharing)
n = len(qs)
host = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
host.numpy()[:] = qs.positions
qset = fs.QuerySet(host.numpy())
chunks = int(os.environ.get("CHUNKS", "0")) or None
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fs.evaluate_field(cfg, src, kern, qset, tree=tree, chunks=chunks)
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
