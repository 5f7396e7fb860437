"""Loader for the committed golden fixtures (tests/golden/)."""

import functools
import hashlib
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TREE_KEYS = ("bbox_min", "bbox_max", "diameter", "aggregate_mass", "aggregate_weight",
             "center_of_mass", "child_start", "child_count", "child_index", "begin",
             "end", "depth", "permuted_indices", "points", "masses", "weights")


@functools.lru_cache(maxsize=1)
def meta():
    with open(os.path.join(HERE, "golden.json")) as f:
        return json.load(f)


@functools.lru_cache(maxsize=1)
def arrays():
    with np.load(os.path.join(HERE, "golden.npz")) as z:
        return {k: z[k] for k in z.files}


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def case_id(case):
    return "-".join(f"{k}{case[k]}" for k in ("kind", "m", "d", "max_depth", "channels")
                    if k in case)


def parse_sto(run):
    """'sto_d2_S3_rr0_seed11_off0' -> (S, rr, seed, off)."""
    parts = {}
    for tok in run.split("_")[1:]:
        head = tok.rstrip("0123456789")
        parts[head] = int(tok[len(head):])
    return parts["S"], parts["rr"], parts["seed"], parts["off"]
