"""Tree built on rank 0 and broadcast to the other rank (sharding.broadcast_tree):
two processes sharing cuda:0 over gloo (the NCCL path needs one GPU per rank).
The assembled tree evaluates bit-identically to the source rank's.  Needs a GPU."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


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
    from paper_2506_02219_b200.sharding import broadcast_tree
    import scenes
    s = scenes.build_sources(dict(kind="mesh_torus", m=30000, seed=3))
    tree = broadcast_tree(s if rank == 0 else None, 4, src=0)
    kern = fs.KernelSpec("coulomb")
    q = fs.QuerySet(np.random.default_rng(4).uniform(-0.6, 0.6, (5000, 3)))
    res = {}
    for prec in ("f32", "f64"):
        for sharing in ("query", "warp"):
            r = fs.evaluate_field(fs.EstimatorConfig("stochastic", seed=2, precision=prec,
                                                     rng_sharing=sharing), s, kern, q, tree=tree)
            res[f"{prec}_{sharing}"] = r.raw
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


def test_broadcast_tree_equals_source_rank(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    a = np.load(tmp_path / "rank0.npz")
    b = np.load(tmp_path / "rank1.npz")
    for k in a.files:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
