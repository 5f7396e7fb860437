"""World-size-2 gloo test of the query-slab sharding path (CPU, no GPU needed).

Each rank evaluates its slab [start, stop) with query_offset = start; the slabs
are all-gathered and must equal a single-process evaluation bit for bit (the
RNG streams are keyed on global query indices, reference _core.py:219,258).
The per-slab evaluator here is the C oracle (test checker); the GPU path uses
the same slab / offset / gather logic (paper_2506_02219_b200/sharding.py).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2506_02219_b200.sharding import slab


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    import scenes
    s = scenes.make_sources(300, seed=71)
    q = scenes.make_query_points(101, seed=72)
    return s, q


def _oracle_slab(s, q, start, stop):
    from oracle import oracle as O
    t = O.build_tree(s.positions, s.masses, s.weights, 4, 32)
    n = stop - start
    out = np.zeros(n)
    z = [np.zeros(n, dtype=np.int64) for _ in range(3)]
    O.stochastic_batch(*O.core_arrays(t), 0, 200.0, 1e-12, q[start:stop], 2, 0, 13, start, out, *z)
    return out


def _worker(rank, world, port, result_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_2506_02219_b200.sharding import gather_slabs, slab as slab_
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, q = _scene()
    a, b = slab_(len(q), rank, world)
    local = torch.from_numpy(_oracle_slab(s, q, a, b))
    full = gather_slabs(local, len(q))
    if rank == 0:
        np.save(result_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_slab_partition_is_balanced_and_complete():
    for n in (1, 7, 100, 101, 4096):
        for world in (1, 2, 3, 8):
            spans = [slab(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slab(10, 2, 2)


def test_two_rank_gloo_gather_equals_single_process(tmp_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    path = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    gathered = np.load(path)
    s, q = _scene()
    single = _oracle_slab(s, q, 0, len(q))
    np.testing.assert_array_equal(gathered, single)


def test_aligned_slabs_start_on_windows():
    for n in (1, 100, 65536, 200_001, 10 ** 6):
        for world in (1, 2, 3, 8):
            spans = [slab(n, r, world, 1 << 16) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert all(a % (1 << 16) == 0 for a, _ in spans)


def _warp_worker(rank, world, port, result_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2506_02219_b200.sharding import SHUFFLE_WINDOW, gather_slabs, slab as slab_
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, q = _warp_scene()
    a, b = slab_(len(q), rank, world, SHUFFLE_WINDOW)
    local = torch.from_numpy(_oracle_warp_slab(s, q, a, b))
    full = gather_slabs(local, len(q), align=SHUFFLE_WINDOW)
    if rank == 0:
        np.save(result_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _warp_scene():
    import scenes
    s = scenes.make_sources(200, seed=73)
    q = scenes.make_query_points(70_000, seed=74)
    return s, q


def _oracle_warp_slab(s, q, start, stop):
    """The warp-shared mode of one slab: its window-local shuffle keyed on global
    positions (query_offset = start) and group keys (position + offset) >> 5."""
    from oracle import oracle as O
    t = O.build_tree(s.positions, s.masses, s.weights, 4, 32)
    n = stop - start
    out = np.zeros(n)
    z = [np.zeros(n, dtype=np.int64) for _ in range(3)]
    if n:
        O.stochastic_ex_batch(*O.core_arrays(t), 0, 200.0, 1e-12, q[start:stop], 1, 0, 13, start,
                              out, *z, keys=O.shared_keys(n, 13, start))
    return out


def test_two_rank_gloo_warp_shared_streams_equal_single_process(tmp_path):
    """With the paper's shared streams, window-aligned slabs (offset = slab start)
    reproduce the whole set's evaluation bit for bit."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    path = str(tmp_path / "full_warp.npy")
    mp.spawn(_warp_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    gathered = np.load(path)
    s, q = _warp_scene()
    np.testing.assert_array_equal(gathered, _oracle_warp_slab(s, q, 0, len(q)))
