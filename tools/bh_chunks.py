"""Distribution of per-chunk BH work (C4, beta=6): visited counts per 32-query chunk in
the kernel's Morton order, to size the critical path of the warp-union walk."""
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
t2 = fs.build_tree(src, 2)
n = len(qs)
L = _lib.lib()
perm = dev.empty(n, torch.int32)
L.fsb_query_order(C.c_void_p(dev.ptr(q)), n, C.c_void_p(dev.ptr(perm)),
                  C.c_void_p(torch.cuda.current_stream().cuda_stream))
beta = float(os.environ.get("BETA", "6"))
r = evaluate_field_device(fs.EstimatorConfig("barnes_hut", beta=beta, precision="f32"), src, kern, q, t2)
vis = r.visited.cpu().numpy()
order = perm.cpu().numpy()
v = vis[order]
nch = (n + 31) // 32
pad = np.zeros(nch * 32, dtype=np.int64)
pad[:n] = v
ch = pad.reshape(nch, 32)
mx = ch.max(axis=1)
print(f"beta={beta}: queries visited mean {vis.mean():.0f} max {vis.max()} p99 {np.percentile(vis, 99):.0f}")
print(f"chunk max-lane visited: mean {mx.mean():.0f} p99 {np.percentile(mx, 99):.0f} max {mx.max()}")
print(f"sum over chunks of max-lane visited {mx.sum():.3g} (union walk iterations >= this)")
top = np.sort(mx)[::-1][:10]
print("top chunk max-lane visited:", top.tolist())

