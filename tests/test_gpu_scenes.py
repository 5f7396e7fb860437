"""Device input generators (csrc/fs_scene.cu) reproduce the host generators byte for
byte: numpy default_rng PCG64 streams jumped ahead per draw, numpy's choice table,
evaluation order without FMA contraction (scene_io.py:112-148, 188-212)."""

import numpy as np
import pytest

from paper_2506_02219_b200 import scenes as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _torus():
    v, f = S.torus(0.25, 0.06)
    return S.rotate_x(v, 0.7) + np.array([0.1, 0.05, -0.1]), f


@pytest.mark.parametrize("mesh,kind,m,seed,pm", [
    ("torus", "coulomb", 2 ** 16 + 7, 7, None),
    ("sphere", "winding_dipole", 10001, 2, None),
    ("sphere", "smooth_exp", 4099, 11, 1.0),
    ("torus", "coulomb", 1, 0, None),
])
def test_sample_mesh_surface_device_is_byte_identical(mesh, kind, m, seed, pm):
    v, f = _torus() if mesh == "torus" else S.icosphere(3, 0.5)
    host = S.sample_mesh_surface(v, f, m, seed=seed, kernel_kind=kind, point_mass=pm)
    pos, ms, w = S.sample_mesh_surface_device(v, f, m, seed=seed, kernel_kind=kind, point_mass=pm)
    np.testing.assert_array_equal(pos.cpu().numpy(), host.positions)
    np.testing.assert_array_equal(ms.cpu().numpy().reshape(host.masses.shape), host.masses)
    np.testing.assert_array_equal(w.cpu().numpy(), host.weights)


@pytest.mark.parametrize("spec", [
    S.GridSpec("grid3d", resolution=(17, 9, 5)),
    S.GridSpec("grid3d", resolution=(8,), bounds=((-0.3, -2.0, 0.1), (0.7, 1.0, 0.2))),
    S.GridSpec("slice_plane", resolution=(31, 17), origin=(0.1, -0.2, 0.03), extent=0.7),
    S.GridSpec("slice_plane", resolution=(1000, 1000), origin=(0.0, 0.0, 0.03)),
    S.GridSpec("random", count=10007, seed=5, bounds=((-1.0, -0.5, 0.0), (1.0, 0.5, 2.0))),
])
def test_make_queries_device_is_byte_identical(spec):
    np.testing.assert_array_equal(S.make_queries_device(spec).cpu().numpy(),
                                  S.make_queries(spec).positions)
