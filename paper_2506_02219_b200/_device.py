"""Torch plumbing: device buffers and the current CUDA stream (no arithmetic here)."""

from __future__ import annotations

import warnings

import numpy as np


def torch():
    import torch as _t
    return _t


def device():
    t = torch()
    if not t.cuda.is_available():
        from ._lib import FastsumError
        raise FastsumError("paper_2506_02219_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    return t.device("cuda", t.cuda.current_device())


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def to_device(a, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (async from pinned host memory)."""
    t = torch()
    if isinstance(a, t.Tensor):
        x = a
    else:
        with warnings.catch_warnings():  # read-only inputs are only ever read
            warnings.simplefilter("ignore", UserWarning)
            x = t.from_numpy(np.ascontiguousarray(a))
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    return x.to(device(), non_blocking=True).contiguous()


def empty(shape, dtype):
    return torch().empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype):
    return torch().zeros(shape, dtype=dtype, device=device())


def ptr(x) -> int:
    return 0 if x is None else int(x.data_ptr())


def to_host(x) -> np.ndarray:
    return x.cpu().numpy()
