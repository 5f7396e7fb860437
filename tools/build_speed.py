"""C4 tree build: wall time of the public call (host arrays in) vs the C build from
device-resident inputs, per branching factor."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev, _lib  # noqa: E402

src, qs, kern = bench.workload()
L = _lib.lib()
for d in (4, 2):
    fs.build_tree(src, d)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = fs.build_tree(src, d)
    torch.cuda.synchronize()
    api = (time.perf_counter() - t0) * 1e3
    pos, ms, w = (dev.to_device(a) for a in (src.positions, src.masses, src.weights))
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        h = C.c_void_p()
        t0 = time.perf_counter()
        _lib.check(L.fsb_build_tree(C.c_void_p(dev.ptr(pos)), C.c_void_p(dev.ptr(ms)),
                                    C.c_void_p(dev.ptr(w)), len(src), 1, d, 32, C.byref(h),
                                    C.c_void_p(dev.stream_ptr())))
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
        L.fsb_tree_free(h)
    print(f"d={d}: public build_tree {api:.1f} ms (incl. H2D of host arrays), "
          f"C build from device inputs {min(times):.1f} ms", flush=True)
