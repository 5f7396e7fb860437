"""Median relative error of S=1 in FP64 (parity kernel) vs FP32 (production) on C4."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev, _lib  # noqa: E402
from paper_2506_02219_b200.estimators import evaluate_field_device  # noqa: E402

src, qs, kern = bench.workload()
q = dev.to_device(qs.positions)
n = len(qs)
L = _lib.lib()
truth = dev.empty(n, torch.float64)
pts, ms = dev.to_device(src.positions), dev.to_device(src.masses)
_lib.check(L.fsb_brute_force_f32acc64(0, kern.alpha, kern.distance_floor, C.c_void_p(dev.ptr(pts)),
                                       C.c_void_p(dev.ptr(ms)), len(src), 1, C.c_void_p(dev.ptr(q)), n,
                                       C.c_void_p(dev.ptr(truth)), C.c_void_p(dev.stream_ptr())))
th = truth.cpu().numpy()
t4 = fs.build_tree(src, 4)
for prec in ("f32", "f64"):
    for seed in (1, 2, 3):
        r = evaluate_field_device(fs.EstimatorConfig("stochastic", seed=seed, precision=prec), src, kern, q, t4)
        v = r.values.cpu().numpy()
        print(prec, seed, f"median rel err {np.median(np.abs(v - th) / np.abs(th)):.4e}", flush=True)
