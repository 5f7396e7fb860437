"""Host-side scene and query generators (input preparation, not the hot path).

These restate the reference's mesh and query recipes so benchmark and test
inputs are byte-identical to what the reference would be fed:

* ``triangle_areas_normals`` / ``icosphere`` / ``torus`` -- meshes.py:14-114
* ``sample_mesh_surface`` -- scene_io.py:112-148 (area-uniform sampling)
* ``GridSpec`` / ``make_queries`` -- scene_io.py:151-212

Byte-identity with the reference generators is pinned by the input digests
in ``tests/golden/golden.json``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .types import QuerySet, SourceSet

__all__ = ["triangle_areas_normals", "icosphere", "torus", "sample_mesh_surface",
           "GridSpec", "make_queries", "rotate_x", "sample_mesh_surface_device",
           "make_queries_device"]


def triangle_areas_normals(vertices, faces):
    """meshes.py:14-26."""
    v = np.asarray(vertices, dtype=np.float64)
    f = np.asarray(faces, dtype=np.int64)
    a = v[f[:, 1]] - v[f[:, 0]]
    b = v[f[:, 2]] - v[f[:, 0]]
    cross = np.cross(a, b)
    norms = np.linalg.norm(cross, axis=1)
    areas = 0.5 * norms
    unit = np.zeros_like(cross)
    ok = norms > 0
    unit[ok] = cross[ok] / norms[ok, None]
    return areas, unit


def icosphere(subdivisions: int = 3, radius: float = 1.0, center=(0.0, 0.0, 0.0)):
    """meshes.py:29-78: subdivided icosahedron projected to the sphere."""
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    verts = np.array([
        [-1, phi, 0], [1, phi, 0], [-1, -phi, 0], [1, -phi, 0],
        [0, -1, phi], [0, 1, phi], [0, -1, -phi], [0, 1, -phi],
        [phi, 0, -1], [phi, 0, 1], [-phi, 0, -1], [-phi, 0, 1],
    ], dtype=np.float64)
    verts /= np.linalg.norm(verts, axis=1)[:, None]
    faces = np.array([
        [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
        [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
        [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
        [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1],
    ], dtype=np.int64)
    for _ in range(subdivisions):
        cache: dict[tuple[int, int], int] = {}
        pieces = [verts]
        count = [len(verts)]

        def mid(i, j):
            key = (min(i, j), max(i, j))
            got = cache.get(key)
            if got is not None:
                return got
            m = verts[i] + verts[j]
            m /= np.linalg.norm(m)
            pieces.append(m[None, :])
            cache[key] = count[0]
            count[0] += 1
            return cache[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf.extend([[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]])
        verts = np.vstack(pieces)
        faces = np.array(nf, dtype=np.int64)
    return verts * radius + np.asarray(center, dtype=np.float64), faces


def torus(major_radius: float = 0.6, minor_radius: float = 0.08, segments_major: int = 96,
          segments_minor: int = 24, center=(0.0, 0.0, 0.0)):
    """meshes.py:81-114: closed triangulated torus around z."""
    if not (0 < minor_radius < major_radius):
        raise ValueError("need 0 < minor_radius < major_radius")
    if segments_major < 3 or segments_minor < 3:
        raise ValueError("need at least 3 segments in each direction")
    u = 2.0 * np.pi * np.arange(segments_major) / segments_major
    v = 2.0 * np.pi * np.arange(segments_minor) / segments_minor
    uu, vv = np.meshgrid(u, v, indexing="ij")
    ring = major_radius + minor_radius * np.cos(vv)
    verts = np.column_stack([(ring * np.cos(uu)).ravel(), (ring * np.sin(uu)).ravel(),
                             (minor_radius * np.sin(vv)).ravel()])
    i = np.arange(segments_major)[:, None]
    j = np.arange(segments_minor)[None, :]
    a = i * segments_minor + j
    b = ((i + 1) % segments_major) * segments_minor + j
    a2 = i * segments_minor + (j + 1) % segments_minor
    b2 = ((i + 1) % segments_major) * segments_minor + (j + 1) % segments_minor
    f1 = np.stack([a, b, b2], axis=-1)
    f2 = np.stack([a, b2, a2], axis=-1)
    faces = np.stack([f1, f2], axis=2).reshape(-1, 3).astype(np.int64)
    return verts + np.asarray(center, dtype=np.float64), faces


def rotate_x(vertices, angle: float):
    """Rotate vertices about the x axis (used to tilt the C4 torus)."""
    c, s = np.cos(angle), np.sin(angle)
    rot = np.array([[1.0, 0.0, 0.0], [0.0, c, -s], [0.0, s, c]])
    return np.asarray(vertices, dtype=np.float64) @ rot.T


def sample_mesh_surface(vertices, faces, num_samples: int, seed: int,
                        kernel_kind: str = "coulomb", point_mass: float | None = None) -> SourceSet:
    """scene_io.py:112-148: area-uniform surface samples as a SourceSet."""
    if num_samples < 1:
        raise ValueError("num_samples must be >= 1")
    areas, normals = triangle_areas_normals(vertices, faces)
    total_area = float(areas.sum())
    if total_area <= 0:
        raise ValueError("mesh has zero surface area")
    rng = np.random.default_rng(seed)
    tri = rng.choice(len(areas), size=num_samples, p=areas / total_area)
    u = rng.random(num_samples)
    v = rng.random(num_samples)
    flip = u + v > 1
    u[flip] = 1 - u[flip]
    v[flip] = 1 - v[flip]
    f = np.asarray(faces, dtype=np.int64)[tri]
    va = np.asarray(vertices, dtype=np.float64)
    pts = (va[f[:, 0]] * (1 - u - v)[:, None] + va[f[:, 1]] * u[:, None]
           + va[f[:, 2]] * v[:, None])
    w_each = total_area / num_samples
    if kernel_kind == "winding_dipole":
        masses = normals[tri] * w_each
    else:
        m = (1.0 / num_samples) if point_mass is None else float(point_mass)
        masses = np.full(num_samples, m)
    weights = np.full(num_samples, w_each)
    return SourceSet(pts, masses, weights)


@dataclass(frozen=True)
class GridSpec:
    """scene_io.py:151-179: lattice, embedded slice plane, or random cloud."""

    kind: str
    resolution: tuple = (10, 10, 10)
    bounds: tuple = ((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    origin: tuple = (0.0, 0.0, 0.0)
    u_axis: tuple = (1.0, 0.0, 0.0)
    v_axis: tuple = (0.0, 1.0, 0.0)
    extent: float = 1.0
    count: int = 1000
    seed: int = 0

    def __post_init__(self):
        if self.kind not in ("grid3d", "slice_plane", "random"):
            raise ValueError(f"unknown query kind {self.kind!r}")
        if any(r < 1 for r in self.resolution):
            raise ValueError("resolutions must be >= 1")
        if self.kind == "slice_plane":
            u = np.asarray(self.u_axis, dtype=np.float64)
            v = np.asarray(self.v_axis, dtype=np.float64)
            if (abs(np.linalg.norm(u) - 1) > 1e-9 or abs(np.linalg.norm(v) - 1) > 1e-9
                    or abs(u @ v) > 1e-9):
                raise ValueError("slice axes must be orthonormal")
        if self.kind == "random" and self.count < 1:
            raise ValueError("count must be >= 1")


def _axis(lo, hi, r):
    return np.array([(lo + hi) / 2.0]) if r == 1 else np.linspace(lo, hi, r)


def make_queries(spec: GridSpec) -> QuerySet:
    """scene_io.py:188-212 (grid3d is z-fastest, slices are v-major)."""
    lo, hi = np.asarray(spec.bounds[0]), np.asarray(spec.bounds[1])
    if spec.kind == "grid3d":
        res = tuple(spec.resolution)
        rx, ry, rz = (res * 3)[:3] if len(res) == 1 else res[:3]
        gx, gy, gz = np.meshgrid(_axis(lo[0], hi[0], rx), _axis(lo[1], hi[1], ry),
                                 _axis(lo[2], hi[2], rz), indexing="ij")
        return QuerySet(np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()]))
    if spec.kind == "slice_plane":
        res = tuple(spec.resolution)
        nu, nv = (res * 2)[:2] if len(res) == 1 else res[:2]
        su = _axis(-spec.extent, spec.extent, nu)
        sv = _axis(-spec.extent, spec.extent, nv)
        o = np.asarray(spec.origin, dtype=np.float64)
        u = np.asarray(spec.u_axis, dtype=np.float64)
        v = np.asarray(spec.v_axis, dtype=np.float64)
        pts = (o[None, :] + sv[:, None, None] * v[None, None, :]
               + su[None, :, None] * u[None, None, :]).reshape(-1, 3)
        return QuerySet(pts)
    rng = np.random.default_rng(spec.seed)
    return QuerySet(rng.uniform(lo, hi, size=(spec.count, 3)))


# --------------------------------------------------------------------------
# Device generators (csrc/fs_scene.cu): the same bytes, drawn on the GPU
# --------------------------------------------------------------------------

def _pcg_state4(seed):
    """{state_hi, state_lo, inc_hi, inc_lo} of numpy default_rng(seed) before its first draw."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    m64 = (1 << 64) - 1
    s, inc = int(st["state"]), int(st["inc"])
    return np.array([s >> 64, s & m64, inc >> 64, inc & m64], dtype=np.uint64)


def sample_mesh_surface_device(vertices, faces, num_samples: int, seed: int,
                               kernel_kind: str = "coulomb", point_mass: float | None = None):
    """sample_mesh_surface drawn on the GPU: (positions (M,3), masses (M,c), weights (M,))
    as CUDA tensors, byte-identical to the host generator (scene_io.py:112-148)."""
    import ctypes as C
    from . import _device as dev
    from . import _lib
    torch = dev.torch()
    if num_samples < 1:
        raise ValueError("num_samples must be >= 1")
    areas, normals = triangle_areas_normals(vertices, faces)
    total_area = float(areas.sum())
    if total_area <= 0:
        raise ValueError("mesh has zero surface area")
    p = areas / total_area
    cdf = p.cumsum()  # numpy Generator.choice's table (replace=True, p given)
    cdf /= cdf[-1]
    f = np.asarray(faces, dtype=np.int64)
    tri = np.asarray(vertices, dtype=np.float64)[f]  # (F, 3, 3)
    w_each = total_area / num_samples
    wind = kernel_kind == "winding_dipole"
    mass = (1.0 / num_samples) if point_mass is None else float(point_mass)
    d_cdf, d_tri = dev.to_device(cdf), dev.to_device(np.ascontiguousarray(tri))
    d_nrm = dev.to_device(np.ascontiguousarray(normals)) if wind else None
    pos = dev.empty((num_samples, 3), torch.float64)
    ms = dev.empty((num_samples, 3) if wind else (num_samples, 1), torch.float64)
    w = dev.empty(num_samples, torch.float64)
    st = _pcg_state4(seed)
    _lib.check(_lib.lib().fsb_sample_mesh_surface(
        C.c_void_p(dev.ptr(d_cdf)), len(cdf), C.c_void_p(dev.ptr(d_tri)),
        C.c_void_p(dev.ptr(d_nrm)), num_samples, st.ctypes.data_as(C.c_void_p), w_each, mass,
        C.c_void_p(dev.ptr(pos)), C.c_void_p(dev.ptr(ms)), C.c_void_p(dev.ptr(w)),
        C.c_void_p(dev.stream_ptr())))
    dev.torch().cuda.current_stream().synchronize()  # the host arrays above are freed on return
    return pos, ms, w


def make_queries_device(spec: GridSpec):
    """make_queries on the GPU: an (N,3) float64 CUDA tensor with the host bytes."""
    import ctypes as C
    from . import _device as dev
    from . import _lib
    torch = dev.torch()
    lo, hi = np.asarray(spec.bounds[0], dtype=np.float64), np.asarray(spec.bounds[1], dtype=np.float64)
    L = _lib.lib()
    st = None
    if spec.kind == "grid3d":
        res = tuple(spec.resolution)
        rx, ry, rz = (res * 3)[:3] if len(res) == 1 else res[:3]
        axes = [_axis(lo[0], hi[0], rx), _axis(lo[1], hi[1], ry), _axis(lo[2], hi[2], rz)]
        kind, n, r1, r2, geo = 0, rx * ry * rz, ry, rz, None
    elif spec.kind == "slice_plane":
        res = tuple(spec.resolution)
        nu, nv = (res * 2)[:2] if len(res) == 1 else res[:2]
        axes = [_axis(-spec.extent, spec.extent, nu), _axis(-spec.extent, spec.extent, nv),
                None]
        kind, n, r1, r2 = 1, nu * nv, nu, 0
        geo = np.concatenate([np.asarray(spec.origin, dtype=np.float64),
                              np.asarray(spec.u_axis, dtype=np.float64),
                              np.asarray(spec.v_axis, dtype=np.float64)])
    else:
        axes = [None, None, None]
        kind, n, r1, r2 = 2, spec.count, 0, 0
        geo = np.concatenate([lo, hi])
        st = _pcg_state4(spec.seed)
    d_axes = [None if a is None else dev.to_device(a) for a in axes]
    d_geo = None if geo is None else dev.to_device(geo)
    out = dev.empty((n, 3), torch.float64)
    _lib.check(L.fsb_make_queries(
        kind, n, *(C.c_void_p(dev.ptr(a)) for a in d_axes), r1, r2, C.c_void_p(dev.ptr(d_geo)),
        None if st is None else st.ctypes.data_as(C.c_void_p), C.c_void_p(dev.ptr(out)),
        C.c_void_p(dev.stream_ptr())))
    torch.cuda.current_stream().synchronize()
    return out
