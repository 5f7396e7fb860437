"""Writers and parsers of scene_io (reference scene_io.py:39-283) on the host.

Every output file must equal, byte for byte, the file the reference's own
writer produced for the same inputs (tests/golden/io/, made by
tests/golden/make_io_golden.py from the imported reference).  The CSV and
points-file rows are formatted by the native writers in csrc/fs_io.cu (host
code: no GPU needed).
"""

import os

import numpy as np
import pytest

import io_cases
from paper_2506_02219_b200 import scene_io as sio
from paper_2506_02219_b200.estimators import FieldResult
from paper_2506_02219_b200.types import SourceSet

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def _field(case, n):
    vals, flags = io_cases.field_values(case, n)
    z = np.zeros(n, dtype=np.int64)
    return FieldResult(values=vals, raw=vals.copy(), flagged=flags, visited_nodes=z,
                       path_steps=z, path_count=z, method="stochastic")


@pytest.mark.parametrize("name", sorted(io_cases.FIELD_CASES))
def test_write_outputs_bytes_equal_reference(name, tmp_path):
    case = io_cases.FIELD_CASES[name]
    spec = sio.GridSpec(**case["spec"])
    q = sio.make_queries(spec)
    with np.errstate(over="ignore"):
        paths = sio.write_outputs(_field(case, len(q)), q, spec, str(tmp_path / name),
                                  **case.get("kw", {}))
    want = sorted(f for f in os.listdir(GOLD) if f.startswith(name + "."))
    assert sorted(os.path.basename(p) for p in paths.values()) == want
    for f in want:
        assert (tmp_path / f).read_bytes() == open(os.path.join(GOLD, f), "rb").read(), f


@pytest.mark.parametrize("name", sorted(io_cases.POINT_CASES))
def test_points_file_round_trip_bytes_equal_reference(name, tmp_path):
    pos, ms = io_cases.point_arrays(io_cases.POINT_CASES[name])
    path = tmp_path / (name + ".txt")
    sio.write_points_file(path, SourceSet(pos, ms))
    assert path.read_bytes() == open(os.path.join(GOLD, name + ".txt"), "rb").read()
    back = sio.parse_points_file(path)  # %.17g round-trips every double exactly
    np.testing.assert_array_equal(back.positions, pos)
    np.testing.assert_array_equal(back.masses, ms.reshape(len(pos), -1))


def test_csv_writer_large_block_boundaries(tmp_path):
    """Rows cross the native writer's 64 Ki-row blocks in order (and match Python's
    formatting of every row)."""
    n = 3 * (1 << 16) + 17
    rng = np.random.default_rng(0)
    q = sio.QuerySet(rng.uniform(-1, 1, (n, 3)))
    vals = rng.normal(size=n)
    flags = rng.random(n) < 0.01
    z = np.zeros(n, dtype=np.int64)
    res = FieldResult(values=vals, raw=vals, flagged=flags, visited_nodes=z, path_steps=z,
                      path_count=z, method="brute_force")
    sio.write_outputs(res, q, sio.GridSpec("random", count=n), str(tmp_path / "big"))
    lines = (tmp_path / "big.csv").read_text().splitlines()
    assert len(lines) == n + 1
    for i in (0, 1, (1 << 16) - 1, 1 << 16, 2 * (1 << 16) + 5, n - 1):
        x, y, zz = q.positions[i]
        assert lines[i + 1] == f"{i},{x:.17g},{y:.17g},{zz:.17g},{vals[i]:.17g},{int(flags[i])}"


def test_parse_errors_name_the_line(tmp_path):
    p = tmp_path / "bad.txt"
    p.write_text("# header\n1 2 3 4\n1 2 3\n")
    with pytest.raises(sio.PointsFileError, match=r"bad.txt:3: inconsistent column count"):
        sio.parse_points_file(p)
    p.write_text("1 2 3\n")
    with pytest.raises(sio.PointsFileError, match="expected 4 or 6 columns"):
        sio.parse_points_file(p)
    p.write_text("1 2 x 4\n")
    with pytest.raises(sio.PointsFileError, match="non-numeric"):
        sio.parse_points_file(p)
    p.write_text("1 2 inf 4\n")
    with pytest.raises(sio.PointsFileError, match="non-finite"):
        sio.parse_points_file(p)
    p.write_text("# nothing\n\n")
    with pytest.raises(sio.PointsFileError, match="no data lines"):
        sio.parse_points_file(p)


def test_load_obj_fan_triangulates_and_resolves_indices(tmp_path):
    p = tmp_path / "quad.obj"
    p.write_text("# quad\nv 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nvn 0 0 1\nf 1/1/1 2 3 -1\n")
    v, f = sio.load_obj(p)
    assert v.shape == (4, 3) and f.dtype == np.int64
    np.testing.assert_array_equal(f, [[0, 1, 2], [0, 2, 3]])
    p.write_text("v 0 0 0\nf 1 1\n")
    with pytest.raises(sio.PointsFileError, match="face with <3 vertices"):
        sio.load_obj(p)
