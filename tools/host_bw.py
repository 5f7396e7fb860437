"""Host memory bandwidth for the e2e pipeline's host-side column work: memcpy of
8 MB float64 and int32 -> int64 widening, 1..16 threads (numpy releases the GIL)."""
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 1_000_000
src = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
dst = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
s32 = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
d64 = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
src[:] = 1.0
s32[:] = 7
for th in (1, 2, 4, 8, 16):
    ex = ThreadPoolExecutor(th)
    parts = np.array_split(np.arange(n), th)
    rng = [(p[0], p[-1] + 1) for p in parts]

    def cp(r):
        np.copyto(dst[r[0]:r[1]], src[r[0]:r[1]])

    def wd(r):
        np.copyto(d64[r[0]:r[1]], s32[r[0]:r[1]], casting="unsafe")
    for f, name in ((cp, "memcpy f64 8MB"), (wd, "widen i32->i64 4MB->8MB")):
        list(ex.map(f, rng))
        t0 = time.perf_counter()
        for _ in range(20):
            list(ex.map(f, rng))
        dt = (time.perf_counter() - t0) / 20
        print(f"{th:2d} threads {name}: {dt * 1e3:.3f} ms", flush=True)
    ex.shutdown()
