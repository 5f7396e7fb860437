import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2506_02219_b200 as fs
from paper_2506_02219_b200 import _device as dev
from paper_2506_02219_b200.estimators import evaluate_field_device
src, qs, kern = bench.workload()
q = dev.to_device(qs.positions)
t4 = fs.build_tree(src, 4)
cfg = fs.EstimatorConfig("stochastic", seed=1)
for i in range(6):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); evaluate_field_device(cfg, src, kern, q, t4); b.record(); torch.cuda.synchronize()
    print("f64 sto evaluate_field_device", i, a.elapsed_time(b))
