"""Device step time of the FP32 stochastic estimator (both stream modes) on the
secondary configs of tools/configs.py: python tools/sto_time.py C2s C2t C1 C5"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import configs  # noqa: E402
import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _device as dev  # noqa: E402
from paper_2506_02219_b200.estimators import evaluate_field_device  # noqa: E402

for name in sys.argv[1:] or ["C2s", "C2t"]:
    src, qs, kern, _, _ = configs.scene(name)
    q = dev.to_device(qs.positions)
    t4 = fs.build_tree(src, 4)
    for sharing in ("query", "warp"):
        cfg = fs.EstimatorConfig("stochastic", seed=1, precision="f32", rng_sharing=sharing)
        ms, _ = configs.timed(lambda: evaluate_field_device(cfg, src, kern, q, t4), reps=10)
        print(f"{os.environ.get('FSB_LIB', 'default')} {name} {sharing}: {ms:.3f} ms", flush=True)
