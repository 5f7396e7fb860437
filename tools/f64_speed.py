"""C4: device step times of the FP64 parity path (the API default precision) vs FP32."""
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
t4, t2 = fs.build_tree(src, 4), fs.build_tree(src, 2)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for method, tree, extra in (("stochastic", t4, {}), ("barnes_hut", t2, {"beta": 6.0})):
    for prec in ("f32", "f64"):
        cfg = fs.EstimatorConfig(method, precision=prec, **extra)
        evaluate_field_device(cfg, src, kern, q, tree)
        torch.cuda.synchronize()
        a.record()
        for _ in range(3):
            evaluate_field_device(cfg, src, kern, q, tree)
        b.record()
        torch.cuda.synchronize()
        print(f"{method} {prec}: {a.elapsed_time(b) / 3:.2f} ms", flush=True)
