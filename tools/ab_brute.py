"""Time the FP32 brute force (FP64 accumulation) on 2^20 sources x 2^18 queries."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_02219_b200 import _device as dev, _lib  # noqa: E402

rng = np.random.default_rng(0)
m, n = 2 ** 20, 2 ** 18
pts, ms = dev.to_device(rng.uniform(-1, 1, (m, 3))), dev.to_device(np.full(m, 1.0 / m))
q = dev.to_device(rng.uniform(-1, 1, (n, 3)))
out = dev.empty(n, torch.float64)
L = _lib.lib()


def run():
    _lib.check(L.fsb_brute_force_f32acc64(0, 200.0, 1e-12, C.c_void_p(dev.ptr(pts)),
                                           C.c_void_p(dev.ptr(ms)), m, 1, C.c_void_p(dev.ptr(q)), n,
                                           C.c_void_p(dev.ptr(out)), C.c_void_p(dev.stream_ptr())))


run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    run()
b.record()
torch.cuda.synchronize()
ms_ = a.elapsed_time(b) / 5
rate = m * n / (ms_ * 1e-3)
print(f"{os.environ.get('FSB_LIB', 'default')}: {ms_:.2f} ms, {rate:.3e} interactions/s "
      f"({rate / 4.65e12:.3f} of the MUFU.RSQ bound), checksum {out.sum().item():.12e}")
