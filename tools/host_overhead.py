"""Host-side cost per call of the device-resident stochastic step (C4, warp-shared
streams): wall time of enqueueing N calls without synchronising vs their GPU time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev  # noqa: E402
from paper_2506_02219_b200.estimators import evaluate_field_device  # noqa: E402

src, qs, kern = bench.workload()
q = dev.to_device(qs.positions)
t4 = fs.build_tree(src, 4)
cfg = fs.EstimatorConfig("stochastic", seed=1, precision="f32", rng_sharing="warp")
for _ in range(5):
    evaluate_field_device(cfg, src, kern, q, t4)
torch.cuda.synchronize()
N = 50
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a.record()
for _ in range(N):
    evaluate_field_device(cfg, src, kern, q, t4)
t1 = time.perf_counter()
b.record()
torch.cuda.synchronize()
print(f"host enqueue {1e3 * (t1 - t0) / N:.3f} ms/call, GPU {a.elapsed_time(b) / N:.3f} ms/call")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    evaluate_field_device(cfg, src, kern, q, t4)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(3)

# the same back-to-back loop while the bench's clock samplers run
for label, use_nvml, use_smi in (("no sampler", False, False), ("nvml process", True, False),
                                 ("nvidia-smi -lms 50", False, True), ("both", True, True)):
    clk = bench.Clocks(0)
    if not use_nvml:
        bench._NVML_POLLER_SAVE = bench._NVML_POLLER
    import subprocess as sp  # noqa: E402
    procs = []
    if use_nvml:
        procs.append(sp.Popen([sys.executable, "-c", bench._NVML_POLLER, "0"], stdout=sp.DEVNULL))
    if use_smi:
        procs.append(sp.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv",
                               "-lms", "50"], stdout=sp.DEVNULL))
    time.sleep(1.0)
    for rep in range(3):
        torch.cuda.synchronize()
        a.record()
        for _ in range(30):
            evaluate_field_device(cfg, src, kern, q, t4)
        b.record()
        torch.cuda.synchronize()
        print(f"{label}: {a.elapsed_time(b) / 30:.3f} ms/step")
    for p in procs:
        p.terminate()
        p.wait()

# after a torch.profiler (CUPTI) session, as bench.py counts its launches
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    evaluate_field_device(cfg, src, kern, q, t4)
    torch.cuda.synchronize()
for rep in range(4):
    torch.cuda.synchronize()
    a.record()
    for _ in range(30):
        evaluate_field_device(cfg, src, kern, q, t4)
    b.record()
    torch.cuda.synchronize()
    print(f"after torch.profiler: {a.elapsed_time(b) / 30:.3f} ms/step")
