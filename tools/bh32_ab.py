"""The warp-coherent FP32 BH (FSB_BH_SPLIT=0: k_bh<F32>) on C4 at beta 2 and 6.4,
for the library in FSB_LIB: ms per call and a checksum."""
import os
import sys

os.environ["FSB_BH_SPLIT"] = "0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev  # noqa: E402
from paper_2506_02219_b200.estimators import evaluate_field_device  # noqa: E402

src, qs, kern = bench.workload()
t2 = fs.build_tree(src, 2)
q = dev.to_device(qs.positions)
tag = os.path.basename(os.environ.get("FSB_LIB", "default"))
for beta in (2.0, 6.4):
    cfg = fs.EstimatorConfig("barnes_hut", beta=beta, precision="f32")
    for _ in range(2):
        r = evaluate_field_device(cfg, src, kern, q, t2)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        r = evaluate_field_device(cfg, src, kern, q, t2)
    b.record()
    torch.cuda.synchronize()
    print(f"{tag:>10} beta={beta}: {a.elapsed_time(b) / 5:.3f} ms  checksum {r.raw.double().sum().item():.12e}",
          flush=True)
