"""C4: the paper's warp-shared RNG recipe (rng_sharing="warp") vs the reference's
per-query streams: device step time and median relative error vs brute force."""
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
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ("query", "warp"):
    for prec in ("f32",):
        cfg = fs.EstimatorConfig("stochastic", seed=1, precision=prec, rng_sharing=mode)
        for _ in range(3):
            r = evaluate_field_device(cfg, src, kern, q, t4)
        torch.cuda.synchronize()
        a.record()
        for _ in range(10):
            r = evaluate_field_device(cfg, src, kern, q, t4)
        b.record()
        torch.cuda.synchronize()
        errs = []
        for seed in (1, 2, 3):
            rr = evaluate_field_device(fs.EstimatorConfig("stochastic", seed=seed, precision=prec,
                                                          rng_sharing=mode), src, kern, q, t4)
            v = rr.values.cpu().numpy()
            errs.append(float(np.median(np.abs(v - th) / np.abs(th))))
        print(f"{mode:5s} {prec}: {a.elapsed_time(b) / 10:.3f} ms/step, median rel err "
              f"{np.mean(errs):.4e} (seeds 1-3: {', '.join(f'{e:.4e}' for e in errs)}), "
              f"visited mean {r.visited.double().mean().item():.1f}", flush=True)
