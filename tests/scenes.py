"""Deterministic test scenes (inputs only).

``make_sources`` / ``make_query_points`` restate the reference suite's
``tests/_scenes.py:8-21``; the other kinds add the adversarial inputs the
survey calls for (coincident points, depth-capped duplicates, tight clusters,
grid-aligned near-boundary lattices in a non-dyadic box, >= 9-point leaves)
and the mesh scenes of BASELINE.json's configs.  Their bytes are pinned by
the digests in golden/golden.json.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2506_02219_b200 import scenes as S  # noqa: E402
from paper_2506_02219_b200.types import SourceSet  # noqa: E402


def make_sources(m, seed, channels=1, span=1.0):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-span, span, size=(m, 3))
    masses = rng.normal(size=(m, channels))
    return SourceSet(pos, masses)


def make_query_points(n, seed, span=1.5):
    rng = np.random.default_rng(seed)
    return rng.uniform(-span, span, size=(n, 3))


def c4_torus_mesh():
    """torus(0.25, 0.06) tilted 0.7 rad about x, shifted."""
    v, f = S.torus(0.25, 0.06)
    v = S.rotate_x(v, 0.7) + np.array([0.1, 0.05, -0.1])
    return v, f


def _masses(rng, m, channels, posmass):
    ms = rng.normal(size=(m, channels))
    if posmass:
        ms = np.abs(ms) + 0.1
    return ms


def build_sources(case) -> SourceSet:
    kind, m, seed = case["kind"], case["m"], case["seed"]
    ch = case.get("channels", 1)
    posmass = case.get("posmass", False)
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        if posmass:
            s = make_sources(m, seed, ch)
            return SourceSet(s.positions, np.abs(s.masses) + 0.1)
        return make_sources(m, seed, ch)
    if kind == "c1":
        pos = np.random.default_rng(0).uniform(-1, 1, (m, 3))
        return SourceSet(pos, np.full(m, 1.0 / m))
    if kind == "coincident":
        p = rng.uniform(-1, 1, size=3)
        return SourceSet(np.tile(p, (m, 1)), _masses(rng, m, ch, posmass))
    if kind == "duplicates":
        base = rng.uniform(-1, 1, size=(max(2, m // 5), 3))
        pos = base[rng.integers(0, base.shape[0], size=m)]
        return SourceSet(pos, _masses(rng, m, ch, posmass))
    if kind == "manydup":
        base = rng.uniform(-1, 1, size=(-(-m // 12), 3))
        pos = np.repeat(base, 12, axis=0)[:m]
        pos = pos[rng.permutation(m)]
        return SourceSet(pos, _masses(rng, m, ch, posmass))
    if kind == "cluster":
        c = rng.uniform(-0.5, 0.5, size=3)
        pos = c + 1e-6 * rng.normal(size=(m, 3))
        pos[: max(1, m // 20)] = rng.uniform(-1, 1, size=(max(1, m // 20), 3))
        return SourceSet(pos, _masses(rng, m, ch, posmass))
    if kind == "lattice":
        k = int(round(m ** (1.0 / 3.0)))
        g = np.arange(k, dtype=np.float64)
        gx, gy, gz = np.meshgrid(g, g, g, indexing="ij")
        pts = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
        # non-dyadic spacing and an off-centre origin put points on and next
        # to the per-level cell boundaries the FP64 digit recurrence decides
        h = 0.1 + 0.01 * (seed % 7)
        pts = 0.37 + h * pts
        pts = pts[rng.permutation(pts.shape[0])]
        return SourceSet(pts, _masses(rng, pts.shape[0], ch, posmass))
    if kind == "mesh_torus":
        v, f = c4_torus_mesh()
        return S.sample_mesh_surface(v, f, m, seed, "coulomb", case.get("point_mass"))
    if kind == "mesh_sphere_winding":
        v, f = S.icosphere(3, 0.5)
        return S.sample_mesh_surface(v, f, m, seed, "winding_dipole")
    raise ValueError(kind)


def reference_sources(case, fastsum_mod):
    """The same scene through the reference's own generators (golden script only)."""
    kind = case["kind"]
    if kind not in ("mesh_torus", "mesh_sphere_winding"):
        return None
    from fastsum.meshes import icosphere, torus
    from fastsum.scene_io import sample_mesh_surface
    if kind == "mesh_torus":
        v, f = torus(0.25, 0.06)
        v = S.rotate_x(v, 0.7) + np.array([0.1, 0.05, -0.1])
        return sample_mesh_surface(v, f, case["m"], case["seed"], "coulomb", case.get("point_mass"))
    v, f = icosphere(3, 0.5)
    return sample_mesh_surface(v, f, case["m"], case["seed"], "winding_dipole")
