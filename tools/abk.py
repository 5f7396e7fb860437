"""A/B device timing of the C4 hot kernels for one library build (FSB_LIB=<so>).

    FSB_LIB=abx/v1.so KERNELS=warp,fast,f64 python tools/abk.py

warp: fsb_stochastic_batch_ex, warp-shared streams + in-kernel shuffle (k_sto_warp)
fast: fsb_stochastic_batch FP32, per-query streams (k_sto_fast)
f64:  fsb_stochastic_batch FP64 (the parity kernel; the API default precision)
bh64: fsb_barnes_hut_batch FP64 beta=2 (Morton order)
Prints ms/launch (CUDA events, 10 launches after 3 warm-up) and a checksum.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev, _lib  # noqa: E402

src, qs, kern = bench.workload()
L = _lib.lib()
q = dev.to_device(qs.positions)
n = len(qs)
t4 = fs.build_tree(src, 4)
h4 = C.c_void_p(t4._device_tree().handle)
sp = C.c_void_p(dev.stream_ptr())
vp = lambda t: C.c_void_p(dev.ptr(t))  # noqa: E731
S = int(os.environ.get("S", "1"))
out32 = dev.empty(n, torch.float32)
out64 = dev.empty(n, torch.float64)
vis, st, pc = (dev.empty(n, torch.int64) for _ in range(3))
tag = os.path.basename(os.environ.get("FSB_LIB", "default"))


def timed(name, fn, out, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{tag:>14} {name:>5} S={S}: {a.elapsed_time(b) / reps:7.3f} ms  checksum "
          f"{out.double().sum().item():.12e}  visited {vis.sum().item()} steps {st.sum().item()}", flush=True)


ks = os.environ.get("KERNELS", "warp,fast,f64").split(",")
if "warp" in ks:
    timed("warp", lambda: _lib.check(L.fsb_stochastic_batch_ex(
        h4, 0, 200.0, 1e-12, 1, vp(q), n, None, S, 0, 1, 0, 5, 2, vp(out32), vp(vis), vp(st),
        vp(pc), sp)), out32)
if "fast" in ks:
    timed("fast", lambda: _lib.check(L.fsb_stochastic_batch(
        h4, 0, 200.0, 1e-12, 1, vp(q), n, None, S, 0, 1, 0, vp(out32), vp(vis), vp(st), vp(pc),
        sp)), out32)
if "f64" in ks:
    timed("f64", lambda: _lib.check(L.fsb_stochastic_batch(
        h4, 0, 200.0, 1e-12, 0, vp(q), n, None, S, 0, 1, 0, vp(out64), vp(vis), vp(st), vp(pc),
        sp)), out64, reps=3)
if "bh64" in ks:
    t2 = fs.build_tree(src, 2)
    h2 = C.c_void_p(t2._device_tree().handle)
    perm = dev.empty(n, torch.int32)
    L.fsb_query_order(vp(q), n, vp(perm), sp)
    timed("bh64", lambda: _lib.check(L.fsb_barnes_hut_batch(
        h2, 0, 200.0, 1e-12, 0, vp(q), n, vp(perm), 2.0, vp(out64), vp(vis), sp)), out64, reps=3)
