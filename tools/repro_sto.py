import os, sys, ctypes as C
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import bench
import paper_2506_02219_b200 as fs
from paper_2506_02219_b200 import _device as dev, _lib
m = int(os.environ.get("M", str(2**22)))
nq = int(os.environ.get("NQ", "1000000"))
src, qs, kern = bench.workload(m=m)
L = _lib.lib()
q = dev.to_device(qs.positions[:nq])
t4 = fs.build_tree(src, 4)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
raw = dev.empty(nq, torch.float32); vis = dev.empty(nq, torch.int64)
h = C.c_void_p(t4._device_tree().handle)
for i in range(int(os.environ.get("REPS", "1"))):
    _lib.check(L.fsb_stochastic_batch(h, 0, 200.0, 1e-12, 1, C.c_void_p(dev.ptr(q)), nq, None, 1, 0, 1, 0,
                                      C.c_void_p(dev.ptr(raw)), C.c_void_p(dev.ptr(vis)), None, None, sp))
torch.cuda.synchronize()
print("ok", raw.double().sum().item())
