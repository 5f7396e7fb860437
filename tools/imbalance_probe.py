import os, sys, ctypes as C
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench, paper_2506_02219_b200 as fs
from paper_2506_02219_b200 import _device as dev, _lib
from paper_2506_02219_b200.estimators import evaluate_field_device
src, qs, kern = bench.workload()
q = dev.to_device(qs.positions)
t2 = fs.build_tree(src, 2)
n = len(qs)
perm = dev.empty(n, torch.int32)
L = _lib.lib()
L.fsb_query_order(C.c_void_p(dev.ptr(q)), n, C.c_void_p(dev.ptr(perm)), C.c_void_p(torch.cuda.current_stream().cuda_stream))
r = evaluate_field_device(fs.EstimatorConfig("barnes_hut", beta=6.0, precision="f32"), src, kern, q, t2)
vis = r.visited.cpu().numpy()[perm.cpu().numpy()]
ch = vis[: (n // 32) * 32].reshape(-1, 32)
cmax = ch.max(1); cmean = ch.mean(1)
print("visited mean", vis.mean(), "max", vis.max(), "p99", np.percentile(vis, 99))
print("chunk max: mean", cmax.mean(), "max", cmax.max(), "sum", cmax.sum())
slots = 148 * 40
print("avg load per slot", cmax.sum() / slots, "largest chunk", cmax.max())
srt = np.sort(cmax)[::-1]
print("top10 chunks", srt[:10])
# greedy in Morton order vs LPT
import heapq
def makespan(order):
    h = [0.0] * slots
    heapq.heapify(h)
    for c in order:
        x = heapq.heappop(h); heapq.heappush(h, x + c)
    return max(h)
print("makespan morton", makespan(cmax), "lpt", makespan(srt), "ideal", cmax.sum()/slots)
