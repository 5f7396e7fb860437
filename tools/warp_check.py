"""C4: the warp-uniform shared-stream kernel (k_sto_warp) against k_sto_fast in the
same rng_sharing="warp" mode (FSB_STO_WARP_OFF=1): per-query agreement, walk
counters, step time and median error vs brute force."""
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
ev = torch.cuda.Event
res = {}
for name, off in (("fast", "1"), ("warp", None)):
    if off:
        os.environ["FSB_STO_WARP_OFF"] = off
    else:
        os.environ.pop("FSB_STO_WARP_OFF", None)
    for S in (1, 4):
        cfg = fs.EstimatorConfig("stochastic", seed=1, precision="f32", rng_sharing="warp",
                                 samples_per_subdomain=S)
        for _ in range(3):
            r = evaluate_field_device(cfg, src, kern, q, t4)
        torch.cuda.synchronize()
        a, b = ev(enable_timing=True), ev(enable_timing=True)
        a.record()
        for _ in range(10):
            r = evaluate_field_device(cfg, src, kern, q, t4)
        b.record()
        torch.cuda.synchronize()
        v = r.values.cpu().numpy()
        err = float(np.median(np.abs(v - th) / np.abs(th)))
        res[name, S] = r
        print(f"{name} S={S}: {a.elapsed_time(b) / 10:.3f} ms/step, median rel err {err:.4e}, "
              f"visited {r.visited.double().mean().item():.1f}, steps "
              f"{r.path_steps.double().mean().item():.2f}", flush=True)
for S in (1, 4):
    A, B = res["fast", S], res["warp", S]
    va, vb = A.values.cpu().numpy(), B.values.cpu().numpy()
    rel = np.abs(va - vb) / np.abs(va)
    ds = (A.path_steps != B.path_steps).sum().item()
    dv = (A.visited != B.visited).sum().item()
    print(f"S={S}: max rel diff {rel.max():.3e}, median {np.median(rel):.3e}, "
          f"path_steps differ on {ds} queries, visited on {dv}")
