"""File formats of the reference's scene_io (scene_io.py:1-283), same bytes.

* points files (``x y z m`` or ``x y z mx my mz``, ``#`` comments) and the OBJ
  subset (``v`` / fan-triangulated ``f``) are parsed on the host, with the
  reference's error messages (scene_io.py:39-109);
* ``write_points_file`` and the field CSV of ``write_outputs`` are formatted by
  the native writers in csrc/fs_io.cu (``fsb_write_points_file`` /
  ``fsb_write_field_csv``: Python's ``{:.17g}`` byte for byte, on all host
  threads instead of a Python loop: the 10^6-row C4 plane in tens of ms);
* slice planes get the PFM float map, the 8-bit PGM preview and the JSON
  sidecar (scene_io.py:215-283), vectorised numpy;
* the generators ``sample_mesh_surface`` / ``GridSpec`` / ``make_queries`` live
  in ``scenes`` and are re-exported here under the reference's module name.
"""

from __future__ import annotations

import json
import os

import numpy as np

from . import _lib
from .scenes import GridSpec, make_queries, sample_mesh_surface
from .types import QuerySet, SourceSet

__all__ = ["PointsFileError", "parse_points_file", "write_points_file", "load_obj",
           "sample_mesh_surface", "GridSpec", "make_queries", "write_outputs"]


class PointsFileError(ValueError):
    """Malformed points or OBJ file; the message names the offending line."""


def parse_points_file(path) -> SourceSet:
    """scene_io.py:43-72: 4 or 6 numeric columns, consistent across lines."""
    rows, ncols = [], None
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            body = line.split("#", 1)[0].strip()
            if not body:
                continue
            cols = body.split()
            if ncols is None:
                if len(cols) not in (4, 6):
                    raise PointsFileError(
                        f"{path}:{lineno}: expected 4 or 6 columns, got {len(cols)}")
                ncols = len(cols)
            elif len(cols) != ncols:
                raise PointsFileError(f"{path}:{lineno}: inconsistent column count "
                                      f"({len(cols)} vs {ncols})")
            try:
                vals = [float(c) for c in cols]
            except ValueError:
                raise PointsFileError(f"{path}:{lineno}: non-numeric value") from None
            if not np.all(np.isfinite(vals)):
                raise PointsFileError(f"{path}:{lineno}: non-finite value")
            rows.append(vals)
    if not rows:
        raise PointsFileError(f"{path}: no data lines")
    a = np.array(rows, dtype=np.float64)
    return SourceSet(a[:, :3], a[:, 3:])


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def write_points_file(path, sources: SourceSet) -> None:
    """scene_io.py:75-80, formatted natively (fsb_write_points_file)."""
    pos = np.ascontiguousarray(sources.positions, dtype=np.float64)
    ms = np.ascontiguousarray(sources.masses, dtype=np.float64)
    _lib.check(_lib.load().fsb_write_points_file(_path(path), pos.shape[0], ms.shape[1],
                                                 pos.ctypes.data, ms.ctypes.data))


def load_obj(path):
    """scene_io.py:83-109: vertices (V,3) float64, triangles (F,3) int64."""
    verts, faces = [], []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            parts = line.split()
            if not parts:
                continue
            if parts[0] == "v":
                if len(parts) < 4:
                    raise PointsFileError(f"{path}:{lineno}: bad vertex record")
                verts.append([float(x) for x in parts[1:4]])
            elif parts[0] == "f":
                idx = []
                for tok in parts[1:]:
                    i = int(tok.split("/", 1)[0])
                    idx.append(i - 1 if i > 0 else len(verts) + i)  # 1-based; negative from end
                if len(idx) < 3:
                    raise PointsFileError(f"{path}:{lineno}: face with <3 vertices")
                faces.extend([idx[0], idx[k], idx[k + 1]] for k in range(1, len(idx) - 1))
    if not verts or not faces:
        raise PointsFileError(f"{path}: no usable v/f records")
    return np.array(verts, dtype=np.float64), np.array(faces, dtype=np.int64)


def _write_pfm(path, values2d: np.ndarray) -> None:
    """Pf grayscale, scale -1 (little-endian), rows as stored (scene_io.py:215-221)."""
    h, w = values2d.shape
    with open(path, "wb") as fh:
        fh.write(f"Pf\n{w} {h}\n-1.0\n".encode("ascii"))
        fh.write(np.ascontiguousarray(values2d, dtype="<f4").tobytes())


def _write_pgm(path, values2d: np.ndarray, sentinel2d: np.ndarray, value_range=None):
    """8-bit preview over the finite range, sentinels black (scene_io.py:224-243)."""
    h, w = values2d.shape
    finite = values2d[~sentinel2d]
    if value_range is not None:
        vmin, vmax = float(value_range[0]), float(value_range[1])
    elif finite.size:
        vmin, vmax = float(finite.min()), float(finite.max())
    else:
        vmin = vmax = 0.0
    if vmax > vmin:
        gray = np.clip(np.rint((values2d - vmin) / (vmax - vmin) * 255.0), 0, 255)
        gray = gray.astype(np.uint8)
    else:
        gray = np.full(values2d.shape, 128, dtype=np.uint8)
    gray[sentinel2d] = 0
    with open(path, "wb") as fh:
        fh.write(f"P5\n{w} {h}\n255\n".encode("ascii"))
        fh.write(gray.tobytes())
    return vmin, vmax


def write_outputs(result, queries: QuerySet, spec: GridSpec, out_prefix: str,
                  value_range=None) -> dict:
    """scene_io.py:246-283: the CSV always; slice planes add PFM, PGM and JSON."""
    n = len(queries)
    values = np.ascontiguousarray(result.values, dtype=np.float64)
    if values.shape[0] != n:
        raise ValueError("field length does not match query count")
    flagged = np.ascontiguousarray(result.flagged, dtype=bool)
    q = np.ascontiguousarray(queries.positions, dtype=np.float64)
    paths = {}
    csv_path = f"{out_prefix}.csv"
    _lib.check(_lib.load().fsb_write_field_csv(_path(csv_path), n, q.ctypes.data,
                                               values.ctypes.data, flagged.ctypes.data))
    paths["csv"] = csv_path
    if spec.kind == "slice_plane":
        res = tuple(spec.resolution)
        nu, nv = (res * 2)[:2] if len(res) == 1 else res[:2]
        vals = values.reshape(nv, nu)
        sent = flagged.reshape(nv, nu)
        shown = np.where(sent, 0.0, vals)
        paths["pfm"] = f"{out_prefix}.pfm"
        _write_pfm(paths["pfm"], shown)
        paths["pgm"] = f"{out_prefix}.pgm"
        vmin, vmax = _write_pgm(paths["pgm"], shown, sent, value_range)
        paths["json"] = f"{out_prefix}.json"
        with open(paths["json"], "w", encoding="utf-8") as fh:
            json.dump({"flagged_count": int(sent.sum()), "value_min": vmin, "value_max": vmax,
                       "width": int(nu), "height": int(nv)}, fh, indent=2, sort_keys=True)
            fh.write("\n")
    return paths
