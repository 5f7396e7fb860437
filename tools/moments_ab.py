"""stochastic_moments_batch timing (acceptance criterion 3's shape: 64 queries x
10^5 repetitions) for the library in FSB_LIB; prints ms and a checksum."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_02219_b200 as fs  # noqa: E402
from paper_2506_02219_b200 import _core  # noqa: E402
import scenes  # noqa: E402

tag = os.path.basename(os.environ.get("FSB_LIB", "default"))
s = scenes.build_sources(dict(kind="mesh_torus", m=2 ** 16, seed=3))
tree = fs.build_tree(s, 4)
q = np.random.default_rng(2).uniform(-0.6, 0.6, (64, 3))
for n_reps in (1000, 100_000):
    mean, var = np.zeros(64), np.zeros(64)
    _core.stochastic_moments_batch(*tree.core_arrays(), 0, 200.0, 1e-12, q, 10, 0, np.uint64(5), mean, var)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _core.stochastic_moments_batch(*tree.core_arrays(), 0, 200.0, 1e-12, q, n_reps, 0, np.uint64(5),
                                   mean, var)
    torch.cuda.synchronize()
    print(f"{tag:>8} reps={n_reps}: {1e3 * (time.perf_counter() - t0):9.1f} ms  checksum "
          f"{mean.sum():.17e} {var.sum():.17e}", flush=True)
