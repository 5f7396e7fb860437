"""Where the first build_tree call's time goes (fresh process, C4 scene): CUDA
context, the sources' host->device copy, module loading of the build kernels,
memory-pool growth.  Each phase is timed separately in a fresh process."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
t0 = time.perf_counter()
import torch  # noqa: E402

torch.cuda.init()
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
t1 = time.perf_counter()
import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _lib  # noqa: E402
from paper_2506_02219_b200.octree import device_sources  # noqa: E402

_lib.lib()
t2 = time.perf_counter()
src, qs, kern = bench.workload()
t3 = time.perf_counter()
device_sources(src)
torch.cuda.synchronize()
t4 = time.perf_counter()
t = fs.build_tree(src, 4)
torch.cuda.synchronize()
t5 = time.perf_counter()
del t
t = fs.build_tree(src, 4)
torch.cuda.synchronize()
t6 = time.perf_counter()
print(f"context {1e3*(t1-t0):.0f} ms | library load {1e3*(t2-t1):.0f} ms | scene {1e3*(t3-t2):.0f} ms | "
      f"sources H2D {1e3*(t4-t3):.1f} ms | first build {1e3*(t5-t4):.1f} ms | second build {1e3*(t6-t5):.1f} ms",
      flush=True)
