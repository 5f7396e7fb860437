"""Where the time of a warm build_tree goes (C4 scene): wall time, GPU time, cProfile."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402

src, qs, kern = bench.workload()
for d in (4, 4, 4, 2, 2):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    t = fs.build_tree(src, d)
    b.record()
    torch.cuda.synchronize()
    print(f"d={d}: wall {1e3 * (time.perf_counter() - t0):.2f} ms, events {a.elapsed_time(b):.2f} ms",
          flush=True)
    del t
pr = cProfile.Profile()
pr.enable()
t = fs.build_tree(src, 4)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(12)
