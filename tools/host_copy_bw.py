"""Host-side copy / widen bandwidth on pinned memory (1 and 4 threads): can the
host pipeline replace PCIe bytes by host work?"""
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 1_000_000
src = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy(); src[:] = np.random.rand(n)
dst = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy(); dst[:] = 0
s32 = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy(); s32[:] = 7
d64 = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy(); d64[:] = 0
pool = ThreadPoolExecutor(8)


def timeit(fn, reps=20):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


for th in (1, 2, 4, 8):
    parts = np.array_split(np.arange(n), th)
    sl = [slice(p[0], p[-1] + 1) for p in parts]
    cp = lambda: list(pool.map(lambda s: np.copyto(dst[s], src[s]), sl))  # noqa: E731
    wd = lambda: list(pool.map(lambda s: np.copyto(d64[s], s32[s]), sl))  # noqa: E731
    print(f"threads {th}: copy 8 MB {timeit(cp):.3f} ms, widen int32->int64 (4->8 MB) {timeit(wd):.3f} ms",
          flush=True)
