"""Run the C4 hot-path kernels a few times for ncu (no timing is reported here)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200.estimators import evaluate_field_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="sto,bh")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--beta", type=float, default=6.0)
args = ap.parse_args()
src, qs, kern = bench.workload()
q = fs._device.to_device(qs.positions) if hasattr(fs, "_device") else None
from paper_2506_02219_b200 import _device as dev  # noqa: E402
q = dev.to_device(qs.positions)
t4 = fs.build_tree(src, 4)
t2 = fs.build_tree(src, 2) if "bh" in args.what else None
for _ in range(args.reps):
    if "sto" in args.what:
        evaluate_field_device(fs.EstimatorConfig("stochastic", seed=1, precision="f32"), src, kern, q, t4)
    if "bh" in args.what:
        evaluate_field_device(fs.EstimatorConfig("barnes_hut", beta=args.beta, precision="f32"), src, kern, q, t2)
torch.cuda.synchronize()
print("done")
