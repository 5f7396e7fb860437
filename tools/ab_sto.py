"""A/B timing of the C4 stochastic kernel for alternative builds (FSB_LIB=<so>)."""
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
t4 = fs.build_tree(src, 4)
n = len(qs)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
perm = dev.empty(n, torch.int32)
L.fsb_query_order(C.c_void_p(dev.ptr(q)), n, C.c_void_p(dev.ptr(perm)), sp)
PERM = None if os.environ.get("NOPERM") else C.c_void_p(dev.ptr(perm))
raw = dev.empty(n, torch.float32)
vis = dev.empty(n, torch.int64)
h = C.c_void_p(t4._device_tree().handle)
S = int(os.environ.get("S", "1"))


def run():
    _lib.check(L.fsb_stochastic_batch(h, 0, 200.0, 1e-12, 1, C.c_void_p(dev.ptr(q)), n,
                                      PERM, S, 0, 1, 0,
                                      C.c_void_p(dev.ptr(raw)), C.c_void_p(dev.ptr(vis)), None,
                                      None, sp))


for _ in range(3):
    run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    run()
b.record()
torch.cuda.synchronize()
print(f"{os.environ.get('FSB_LIB', 'default')}{' noperm' if PERM is None else ''}: S={S} {a.elapsed_time(b) / 10:.3f} ms/launch, "
      f"checksum {raw.double().sum().item():.9e}")
