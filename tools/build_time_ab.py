"""C4 tree build from device-resident inputs for the library in FSB_LIB: min of 5
warm builds per branching factor, and a digest of the tree (bitwise comparison
across builds)."""
import ctypes as C
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev, _lib  # noqa: E402

src, qs, kern = bench.workload()
L = _lib.lib()
tag = os.path.basename(os.environ.get("FSB_LIB", "default"))
pos, ms, w = (dev.to_device(a) for a in (src.positions, src.masses, src.weights))
for d in (4, 2):
    t = fs.build_tree(src, d)
    h = hashlib.sha256()
    for k in ("child_start", "child_count", "begin", "end", "permuted_indices", "center_of_mass",
              "aggregate_mass", "diameter"):
        h.update(np.ascontiguousarray(getattr(t, k)).tobytes())
    times = []
    for _ in range(6):
        hh = C.c_void_p()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(L.fsb_build_tree(C.c_void_p(dev.ptr(pos)), C.c_void_p(dev.ptr(ms)),
                                    C.c_void_p(dev.ptr(w)), len(src), 1, d, 32, C.byref(hh),
                                    C.c_void_p(dev.stream_ptr())))
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
        L.fsb_tree_free(hh)
    print(f"{tag:>10} d={d}: {min(times[1:]):.2f} ms (median {np.median(times[1:]):.2f})  "
          f"digest {h.hexdigest()[:16]}", flush=True)
