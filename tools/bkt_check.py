"""Bucketed per-query-stream path vs k_sto_fast (FSB_STO_BUCKET=1 opts in): bitwise
comparison of values and counters, and device time per launch.

    python tools/bkt_check.py [C4 C1 C2s C2t C3] (S=<samples>, RR=<mode>)
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev, _lib  # noqa: E402
from paper_2506_02219_b200.kernels import kernel_id  # noqa: E402

L = _lib.lib()
vp = lambda t: C.c_void_p(dev.ptr(t))  # noqa: E731
S = int(os.environ.get("S", "1"))
RR = int(os.environ.get("RR", "0"))


def scene(name):
    if name == "C4":
        src, qs, kern = bench.workload()
        return src, qs, kern
    import configs
    src, qs, kern, _, _ = configs.scene(name)
    return src, qs, kern


for name in sys.argv[1:] or ["C4"]:
    src, qs, kern = scene(name)
    q = dev.to_device(qs.positions)
    n = len(qs)
    t4 = fs.build_tree(src, 4)
    h = C.c_void_p(t4._device_tree().handle)
    sp = C.c_void_p(dev.stream_ptr())
    kid = kernel_id(kern)
    res = {}
    for mode in ("fast", "bucket"):
        if mode == "fast":
            os.environ.pop("FSB_STO_BUCKET", None)
        else:
            os.environ["FSB_STO_BUCKET"] = "1"
        out = dev.empty(n, torch.float32)
        vis, st, pc = (dev.empty(n, torch.int64) for _ in range(3))

        def run():
            _lib.check(L.fsb_stochastic_batch(h, kid, kern.alpha, kern.distance_floor, 1, vp(q), n,
                                              None, S, RR, 1, 0, vp(out), vp(vis), vp(st), vp(pc),
                                              sp))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        res[mode] = [x.cpu().numpy() for x in (out, vis, st, pc)]
        print(f"{name} S={S} rr={RR} {mode:>6}: {ms:.3f} ms/launch", flush=True)
    f, bk = res["fast"], res["bucket"]
    for lab, x, y in zip(("values", "visited", "steps", "count"), f, bk):
        neq = int(np.sum(x.view(np.uint32 if x.dtype == np.float32 else np.uint64)
                         != y.view(np.uint32 if y.dtype == np.float32 else np.uint64)))
        extra = ""
        if neq and lab == "values":
            d = np.abs(x.astype(np.float64) - y) / (1 + np.abs(x.astype(np.float64)))
            extra = f" max rel {d.max():.3e}"
        print(f"   {lab}: {neq} / {n} differ{extra}", flush=True)
