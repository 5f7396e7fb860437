"""Query-slab sharding through the real CUDA path (sharding.evaluate_field_sharded):
two processes sharing cuda:0 over gloo, each evaluating its slab with the device
kernels and all-gathering the field, against one process evaluating every query
(reference stochastic_batch keys its streams on global query indices,
_core.py:219,258).  The stochastic estimator (both stream modes, FP32 and FP64)
and the FP64 Barnes-Hut are bitwise slab-invariant; the load-balanced FP32
Barnes-Hut sums each query's node set in an order that depends on its warp's
neighbours (fs_bh_split.cu), so it agrees to FP64 rounding.  Needs a GPU."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = {
    "sto_f32_query": dict(method="stochastic", seed=5, precision="f32"),
    "sto_f32_warp": dict(method="stochastic", seed=5, precision="f32", rng_sharing="warp"),
    "sto_f64_query": dict(method="stochastic", seed=5),
    "bh_f64": dict(method="barnes_hut", beta=2.0),
    "bh_f32": dict(method="barnes_hut", beta=4.0, precision="f32"),
}
N_QUERIES = 140_000  # three 2^16 shuffle windows: the warp-shared slabs are window-aligned


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2506_02219_b200 as fs
    from paper_2506_02219_b200.sharding import evaluate_field_sharded, slab
    import scenes
    src = scenes.build_sources(dict(kind="mesh_torus", m=200_000, seed=11))
    q = fs.QuerySet(np.random.default_rng(12).uniform(-0.6, 0.6, (N_QUERIES, 3)))
    kern = fs.KernelSpec("coulomb")
    res = {}
    for name, kw in CASES.items():
        cfg = fs.EstimatorConfig(**kw)
        res[name] = evaluate_field_sharded(cfg, src, kern, q)  # replica tree per rank
        if rank == 0:  # one process, every query
            res[name + "_single"] = fs.evaluate_field(cfg, src, kern, q).values
    res["slab"] = np.array(slab(N_QUERIES, rank, world))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_field_equals_single_process(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    assert tuple(r0["slab"]) == (0, N_QUERIES // 2) and tuple(r1["slab"])[1] == N_QUERIES
    for name in CASES:
        np.testing.assert_array_equal(r0[name], r1[name], err_msg=f"{name}: ranks disagree")
        got, ref = r0[name], r0[name + "_single"]
        assert np.all(np.isfinite(got)), name
        if name == "bh_f32":
            np.testing.assert_allclose(got, ref, rtol=1e-12, atol=0, err_msg=name)
        else:
            np.testing.assert_array_equal(got, ref, err_msg=f"{name}: sharded != single process")
