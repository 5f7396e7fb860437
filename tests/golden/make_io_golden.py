"""Golden output files of the reference's writers (scene_io.py:75-80, 215-283).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_io_golden.py

Each case feeds the reference's ``write_outputs`` / ``write_points_file`` a
FieldResult / SourceSet built from seeded numpy data that exercises the
formatter (negative zero, subnormal and huge magnitudes, integers, +inf flagged
sentinels, a single-resolution slice), and stores the files it writes under
tests/golden/io/<case>.<ext>.  tests/test_scene_io.py rebuilds the same inputs
and requires byte-identical files from paper_2506_02219_b200.scene_io.
"""

from __future__ import annotations

import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
sys.path.insert(0, os.path.dirname(HERE))

import io_cases  # noqa: E402  (the shared case definitions)


def main():
    import fastsum  # the reference, via PYTHONPATH
    from fastsum.estimators import FieldResult
    from fastsum.scene_io import GridSpec, make_queries, write_outputs, write_points_file
    from fastsum.types import SourceSet

    assert "reference" in os.path.dirname(fastsum.__file__), fastsum.__file__
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    for name, case in io_cases.FIELD_CASES.items():
        spec = GridSpec(**case["spec"])
        q = make_queries(spec)
        vals, flags = io_cases.field_values(case, len(q))
        res = FieldResult(values=vals, raw=vals.copy(), flagged=flags,
                          visited_nodes=np.zeros(len(q), dtype=np.int64),
                          path_steps=np.zeros(len(q), dtype=np.int64),
                          path_count=np.zeros(len(q), dtype=np.int64), method="stochastic")
        write_outputs(res, q, spec, os.path.join(OUT, name), **case.get("kw", {}))
    for name, case in io_cases.POINT_CASES.items():
        pos, ms = io_cases.point_arrays(case)
        write_points_file(os.path.join(OUT, name + ".txt"), SourceSet(pos, ms))
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
