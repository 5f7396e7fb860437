"""Generate the golden parity fixtures from the imported reference package.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every fixture is produced by the reference's own public API / numba cores
(``fastsum.build_tree``, ``fastsum._core.*_batch``, ``fastsum.evaluate_field``,
``fastsum.rng``).  Small cases store full arrays; large cases store SHA-256
digests of the reference's output arrays so the bitwise check stays cheap to
commit.  Inputs are regenerated from numpy ``default_rng`` seeds (PCG64 is
stable across numpy versions) and their digests are stored too, which pins
the input generators in ``tests/scenes.py`` against the reference's.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/ for scenes.py

import fastsum  # noqa: E402  (the reference, via PYTHONPATH)
from fastsum import _core  # noqa: E402
from fastsum.estimators import evaluate_field  # noqa: E402
from fastsum.kernels import kernel_id  # noqa: E402
from fastsum.meshes import icosphere, torus  # noqa: E402
from fastsum.octree import build_tree  # noqa: E402
from fastsum.rng import stream_key, uniform_draw  # noqa: E402
from fastsum.scene_io import GridSpec, make_queries, sample_mesh_surface  # noqa: E402
from fastsum.types import EstimatorConfig, KernelSpec, QuerySet, SourceSet  # noqa: E402

import scenes  # noqa: E402  (our regenerators; pinned by the digests below)

TREE_KEYS = ("bbox_min", "bbox_max", "diameter", "aggregate_mass", "aggregate_weight",
             "center_of_mass", "child_start", "child_count", "child_index", "begin",
             "end", "depth", "permuted_indices", "points", "masses", "weights")


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def source_from_case(case):
    return scenes.build_sources(case)


# ------------------------------------------------------------------ cases
SMALL_TREE_CASES = []
for d in (2, 3, 4):
    for m in (1, 2, 17, 200):
        SMALL_TREE_CASES.append(dict(kind="uniform", m=m, seed=d * 100 + m, channels=1,
                                     d=d, max_depth=32))
SMALL_TREE_CASES += [
    dict(kind="uniform", m=64, seed=9, channels=3, d=2, max_depth=32),
    dict(kind="uniform", m=64, seed=9, channels=3, d=4, max_depth=32),
    dict(kind="coincident", m=5, seed=1, channels=1, d=2, max_depth=32),
    dict(kind="coincident", m=12, seed=2, channels=3, d=4, max_depth=32),
    dict(kind="duplicates", m=300, seed=3, channels=1, d=2, max_depth=5),
    dict(kind="duplicates", m=300, seed=4, channels=1, d=4, max_depth=6),
    dict(kind="duplicates", m=300, seed=5, channels=3, d=3, max_depth=4),
    dict(kind="cluster", m=200, seed=6, channels=1, d=2, max_depth=32),
    dict(kind="cluster", m=200, seed=7, channels=1, d=4, max_depth=32),
    dict(kind="lattice", m=512, seed=8, channels=1, d=2, max_depth=32),
    dict(kind="lattice", m=512, seed=9, channels=1, d=4, max_depth=32),
    dict(kind="lattice", m=343, seed=10, channels=1, d=3, max_depth=32),
    dict(kind="uniform", m=40, seed=11, channels=1, d=2, max_depth=1),
    dict(kind="uniform", m=40, seed=12, channels=1, d=4, max_depth=2),
    dict(kind="manydup", m=200, seed=13, channels=1, d=2, max_depth=32),
    dict(kind="manydup", m=200, seed=14, channels=3, d=4, max_depth=32),
]

LARGE_TREE_CASES = [
    dict(kind="uniform", m=2 ** 14, seed=0, channels=1, d=4, max_depth=32, c1=True),
    dict(kind="uniform", m=2 ** 14, seed=0, channels=1, d=2, max_depth=32, c1=True),
    dict(kind="mesh_torus", m=2 ** 15, seed=7, channels=1, d=4, max_depth=32),
    dict(kind="mesh_torus", m=2 ** 15, seed=7, channels=1, d=2, max_depth=32),
    dict(kind="mesh_sphere_winding", m=2 ** 15, seed=2, channels=3, d=4, max_depth=32),
    dict(kind="mesh_sphere_winding", m=2 ** 15, seed=2, channels=3, d=2, max_depth=32),
    dict(kind="lattice", m=32768, seed=21, channels=1, d=4, max_depth=32),
    dict(kind="cluster", m=20000, seed=22, channels=1, d=2, max_depth=32),
]


def ref_tree(case):
    s = source_from_case(case)
    return s, build_tree(s, case["d"], case["max_depth"])


def check_inputs_match(case, s):
    """Our regenerator must produce the reference generator's bytes."""
    ref = scenes.reference_sources(case, fastsum_mod=sys.modules["fastsum"])
    if ref is None:
        return
    for k in ("positions", "masses", "weights"):
        if not np.array_equal(getattr(ref, k), getattr(s, k)):
            raise SystemExit(f"input regenerator mismatch for {case} field {k}")


def main():
    out_arrays = {}
    meta = {"small_trees": [], "large_trees": [], "cores": [], "rng": {}, "f32": []}

    # ---- trees ---------------------------------------------------------
    for ci, case in enumerate(SMALL_TREE_CASES):
        s, t = ref_tree(case)
        check_inputs_match(case, s)
        pre = f"tree{ci}_"
        out_arrays[pre + "in_positions"] = s.positions
        out_arrays[pre + "in_masses"] = s.masses
        out_arrays[pre + "in_weights"] = s.weights
        for k in TREE_KEYS:
            out_arrays[pre + k] = getattr(t, k)
        meta["small_trees"].append(dict(case, prefix=pre, num_nodes=int(t.num_nodes)))
    for case in LARGE_TREE_CASES:
        s, t = ref_tree(case)
        check_inputs_match(case, s)
        entry = dict(case, num_nodes=int(t.num_nodes),
                     inputs={k: digest(getattr(s, k)) for k in ("positions", "masses", "weights")},
                     arrays={k: digest(getattr(t, k)) for k in TREE_KEYS},
                     max_tree_depth=int(t.depth.max()))
        meta["large_trees"].append(entry)
        print("large tree", case, t.num_nodes, int(t.depth.max()), flush=True)

    # ---- cores (f64 parity) -------------------------------------------
    core_cases = [
        dict(src=dict(kind="uniform", m=300, seed=31, channels=1), kernel="coulomb", nq=64),
        dict(src=dict(kind="uniform", m=300, seed=32, channels=3), kernel="winding_dipole", nq=64),
        dict(src=dict(kind="uniform", m=300, seed=33, channels=1, posmass=True),
             kernel="smooth_exp", alpha=20.0, nq=64),
        dict(src=dict(kind="duplicates", m=200, seed=34, channels=1), kernel="coulomb", nq=48,
             max_depth=5),
        dict(src=dict(kind="cluster", m=300, seed=35, channels=1), kernel="coulomb", nq=48),
        dict(src=dict(kind="mesh_torus", m=4096, seed=36, channels=1), kernel="coulomb", nq=128),
        dict(src=dict(kind="mesh_sphere_winding", m=4096, seed=37, channels=3),
             kernel="winding_dipole", nq=128),
        dict(src=dict(kind="uniform", m=1, seed=38, channels=1), kernel="coulomb", nq=8),
        dict(src=dict(kind="coincident", m=6, seed=39, channels=1), kernel="coulomb", nq=8),
    ]
    for k_i, cc in enumerate(core_cases):
        s = scenes.build_sources(cc["src"])
        kern = KernelSpec(cc["kernel"], alpha=cc.get("alpha", 200.0))
        kid = kernel_id(kern)
        qs = scenes.make_query_points(cc["nq"], seed=5000 + k_i)
        pre = f"core{k_i}_"
        out_arrays[pre + "positions"] = s.positions
        out_arrays[pre + "masses"] = s.masses
        out_arrays[pre + "weights"] = s.weights
        out_arrays[pre + "queries"] = qs
        entry = dict(cc, prefix=pre, runs=[])
        # brute force
        o = np.zeros(len(qs))
        _core.brute_force_batch(kid, kern.alpha, kern.distance_floor, s.positions, s.masses, qs, o)
        out_arrays[pre + "brute"] = o
        md = cc.get("max_depth", 32)
        for d in (2, 4):
            t = build_tree(s, d, md)
            ca = t.core_arrays()
            for beta in (0.5, 1.0, 2.0, 4.0, 1e9):
                o = np.zeros(len(qs))
                v = np.zeros(len(qs), dtype=np.int64)
                _core.barnes_hut_batch(*ca, kid, kern.alpha, kern.distance_floor, qs, beta,
                                       (md + 2) * d ** 3 + 8, o, v)
                tag = f"bh_d{d}_b{beta:g}"
                out_arrays[pre + tag] = o
                out_arrays[pre + tag + "_visited"] = v
                entry["runs"].append(tag)
            o = np.zeros(len(qs))
            v = np.zeros(len(qs), dtype=np.int64)
            _core.telescoping_batch(*ca, kid, kern.alpha, kern.distance_floor, qs, o, v)
            tag = f"tel_d{d}"
            out_arrays[pre + tag] = o
            out_arrays[pre + tag + "_visited"] = v
            entry["runs"].append(tag)
            for (S, rr, seed, qoff) in ((1, 0, 0, 0), (3, 0, 11, 0), (2, 1, 5, 17),
                                        (1, 2, 2 ** 64 - 1, 3)):
                o = np.zeros(len(qs))
                v, st, pc = (np.zeros(len(qs), dtype=np.int64) for _ in range(3))
                _core.stochastic_batch(*ca, kid, kern.alpha, kern.distance_floor, qs, S, rr,
                                       np.uint64(seed), qoff, o, v, st, pc)
                tag = f"sto_d{d}_S{S}_rr{rr}_seed{seed}_off{qoff}"
                out_arrays[pre + tag] = o
                out_arrays[pre + tag + "_visited"] = v
                out_arrays[pre + tag + "_steps"] = st
                out_arrays[pre + tag + "_count"] = pc
                entry["runs"].append(tag)
            mean = np.zeros(len(qs))
            var = np.zeros(len(qs))
            _core.stochastic_moments_batch(*ca, kid, kern.alpha, kern.distance_floor, qs, 50, 0,
                                           np.uint64(7), mean, var)
            tag = f"mom_d{d}"
            out_arrays[pre + tag + "_mean"] = mean
            out_arrays[pre + tag + "_var"] = var
            entry["runs"].append(tag)
        meta["cores"].append(entry)
        print("core case", k_i, flush=True)

    # ---- reference precision="f32" runs (for the GPU f32 path) ---------
    f32_cases = [
        dict(src=dict(kind="uniform", m=2000, seed=41, channels=1), kernel="coulomb", nq=256),
        dict(src=dict(kind="mesh_sphere_winding", m=4096, seed=42, channels=3),
             kernel="winding_dipole", nq=256),
        dict(src=dict(kind="mesh_torus", m=4096, seed=43, channels=1, point_mass=1.0),
             kernel="smooth_exp", alpha=50.0, nq=256),
    ]
    for f_i, fc in enumerate(f32_cases):
        s = scenes.build_sources(fc["src"])
        kern = KernelSpec(fc["kernel"], alpha=fc.get("alpha", 200.0))
        qs = scenes.make_query_points(fc["nq"], seed=6000 + f_i)
        pre = f"f32_{f_i}_"
        out_arrays[pre + "queries"] = qs
        entry = dict(fc, prefix=pre, runs=[])
        for method, extra in (("brute_force", {}), ("barnes_hut", dict(beta=2.0)),
                              ("barnes_hut", dict(beta=4.0)),
                              ("stochastic", dict(seed=3)),
                              ("stochastic", dict(seed=3, samples_per_subdomain=4))):
            for prec in ("f32", "f64"):
                r = evaluate_field(EstimatorConfig(method, precision=prec, **extra), s, kern,
                                   QuerySet(qs))
                tag = f"{method}_{'_'.join(f'{k}{v}' for k, v in extra.items())}_{prec}"
                out_arrays[pre + tag + "_raw"] = r.raw
                out_arrays[pre + tag + "_values"] = r.values
                out_arrays[pre + tag + "_visited"] = r.visited_nodes
                entry["runs"].append(tag)
        meta["f32"].append(entry)

    # ---- rng -----------------------------------------------------------
    keys = []
    for args in ((0, 0, 0, 0, 0), (7, 123, 4, 9, 1), (2 ** 64 - 1, 2 ** 40, 63, 255, 0),
                 (12345, 999999, 17, 3, 1)):
        k = int(stream_key(np.uint64(args[0]), args[1], args[2], args[3], args[4]))
        draws = [float(uniform_draw(np.uint64(k), np.uint64(c))) for c in range(8)]
        draws.append(float(uniform_draw(np.uint64(k), np.uint64(2 ** 64 - 1))))
        keys.append(dict(args=[str(a) for a in args], key=str(k), draws=draws))
    meta["rng"]["keys"] = keys

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out_arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(out_arrays), "arrays")


if __name__ == "__main__":
    main()
