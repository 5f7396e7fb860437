"""Timing of the generic FP64 kernels through the device path (FSB_LIB=<so>):
brute force, telescoping, the Alg. 2 stochastic variant, BH (C4 scene, 10^5 / 10^6
queries); prints ms and a checksum per kernel."""
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
tag = os.path.basename(os.environ.get("FSB_LIB", "default"))
t4, t2 = fs.build_tree(src, 4), fs.build_tree(src, 2)
q6 = dev.to_device(qs.positions)
q5 = dev.to_device(qs.positions[::10].copy())
q3 = dev.to_device(qs.positions[::1000].copy())
cases = [
    ("brute", fs.EstimatorConfig("brute_force"), q3, None),
    ("telesc", fs.EstimatorConfig("telescoping_exhaustive", branching_per_dim=4), q3, t4),
    ("alg2", fs.EstimatorConfig("stochastic", seed=1, path_order="roulette_then_swap"), q6, t4),
    ("bh", fs.EstimatorConfig("barnes_hut", beta=2.0), q6, t2),
]
for name, cfg, q, t in cases:
    for _ in range(2):
        r = evaluate_field_device(cfg, src, kern, q, t)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        r = evaluate_field_device(cfg, src, kern, q, t)
    b.record()
    torch.cuda.synchronize()
    print(f"{tag:>10} {name:>7} n={q.shape[0]:>8}: {a.elapsed_time(b) / 3:9.3f} ms  checksum "
          f"{r.raw.double().sum().item():.15e}", flush=True)
