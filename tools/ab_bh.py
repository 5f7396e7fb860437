"""Time the C4 BH kernel (f32) at a few betas via the device API (no truth/error)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev  # noqa: E402
from paper_2506_02219_b200.estimators import evaluate_field_device  # noqa: E402

src, qs, kern = bench.workload()
q = dev.to_device(qs.positions)
t2 = fs.build_tree(src, 2)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
betas = [float(x) for x in os.environ.get("BETAS", "2,6,8").split(",")]
for beta in betas:
    cfg = fs.EstimatorConfig("barnes_hut", beta=beta, precision="f32")
    r = evaluate_field_device(cfg, src, kern, q, t2)
    torch.cuda.synchronize()
    a.record()
    for _ in range(3):
        r = evaluate_field_device(cfg, src, kern, q, t2)
    b.record()
    torch.cuda.synchronize()
    print(f"BH beta={beta}: {a.elapsed_time(b) / 3:.3f} ms, checksum {r.values.sum().item():.9e}, "
          f"visited {r.visited.double().sum().item():.6e}", flush=True)
