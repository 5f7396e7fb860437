"""C4: device time of the stochastic ABI call alone (order precomputed), per-query
streams vs warp-shared streams; FSB_LIB selects a variant library."""
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
q = dev.to_device(qs.positions)
n = len(qs)
L = _lib.lib()
t4 = fs.build_tree(src, 4)
h = C.c_void_p(t4._device_tree().handle)
out = dev.empty(n, torch.float32)
order = dev.empty(n, torch.int32)
sp = C.c_void_p(dev.stream_ptr())
if os.environ.get("ORDER") == "morton":
    _lib.check(L.fsb_query_order(vp(q) if False else C.c_void_p(dev.ptr(q)), n,
                                 C.c_void_p(dev.ptr(order)), sp))
elif os.environ.get("ORDER") == "identity":
    order = torch.arange(n, dtype=torch.int32, device=q.device)
else:
    _lib.check(L.fsb_shuffle_order(n, 1, 0, C.c_void_p(dev.ptr(order)), sp))
vp = lambda t: C.c_void_p(dev.ptr(t))  # noqa: E731
S = int(os.environ.get("S", "1"))


def run(group):
    _lib.check(L.fsb_stochastic_batch_ex(h, 0, kern.alpha, kern.distance_floor, 1, vp(q), n,
                                             vp(order), S, 0, 1, 0, group, 0, vp(out), None, None,
                                             None, sp))


for group, name in ((0, "per-query"), (5, "warp")):
    for _ in range(3):
        run(group)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        run(group)
    b.record()
    torch.cuda.synchronize()
    print(f"{os.environ.get('FSB_LIB', 'default')} {name} S={S} order={os.environ.get('ORDER', 'shuffle')}: "
          f"{a.elapsed_time(b) / 20:.3f} ms")
