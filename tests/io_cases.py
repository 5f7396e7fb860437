"""Inputs of the writer golden cases (tests/golden/make_io_golden.py, test_scene_io.py)."""

from __future__ import annotations

import numpy as np

FIELD_CASES = {
    "slice_7x5": dict(spec=dict(kind="slice_plane", resolution=(7, 5),
                                origin=(0.1, -0.2, 0.03), extent=0.8), seed=1, flag_every=6),
    "slice_sq4": dict(spec=dict(kind="slice_plane", resolution=(4,)), seed=2, flag_every=0),
    "slice_all_flagged": dict(spec=dict(kind="slice_plane", resolution=(3, 2)), seed=3,
                              flag_every=1),
    "slice_range": dict(spec=dict(kind="slice_plane", resolution=(6, 3)), seed=4, flag_every=4,
                        kw=dict(value_range=(-0.5, 0.25))),
    "grid_3": dict(spec=dict(kind="grid3d", resolution=(3, 2, 4)), seed=5, flag_every=0),
    "random_40": dict(spec=dict(kind="random", count=40, seed=9), seed=6, flag_every=7),
}

POINT_CASES = {
    "points_c1": dict(m=37, c=1, seed=11),
    "points_c3": dict(m=23, c=3, seed=12),
}

_SPECIAL = np.array([0.0, -0.0, 1.0, -2.5, 1e-300, 5e-324, 1.7976931348623157e308, 123456789.0,
                     1e16, 1e-5, 0.1, 1.0 / 3.0, -1e22, 2.0 ** 60])


def field_values(case, n):
    rng = np.random.default_rng(case["seed"])
    vals = rng.normal(size=n) * 10.0 ** rng.integers(-8, 9, size=n)
    k = min(n, _SPECIAL.size)
    vals[:k] = _SPECIAL[:k] * (1.0 if case["seed"] % 2 else -1.0)
    flags = np.zeros(n, dtype=bool)
    if case["flag_every"]:
        flags[:: case["flag_every"]] = True
        vals[flags] = np.inf  # smooth_exp sentinel (kernels.py:110-122)
    return vals, flags


def point_arrays(case):
    rng = np.random.default_rng(case["seed"])
    pos = rng.uniform(-1, 1, (case["m"], 3))
    pos[0] = (0.0, -0.0, 1e-310)
    ms = rng.normal(size=(case["m"], case["c"])) * 10.0 ** rng.integers(-5, 6, (case["m"], 1))
    return pos, ms
