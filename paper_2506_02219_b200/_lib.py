"""ctypes binding of libfastsum_b200.so (the C ABI in include/fastsum_b200.h).

There is no CPU fallback: every compute entry point requires the in-tree CUDA
library and a CUDA device, and raises ``RuntimeError`` otherwise.  Device
memory and streams are torch's (plumbing only); all arithmetic runs in the
hand-written sm_100a kernels behind this ABI.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSB_LIB") or os.path.join(_HERE, "libfastsum_b200.so")

_lib = None
_lock = threading.Lock()

_P = C.c_void_p
_I64 = C.c_int64
_I = C.c_int
_D = C.c_double


class EvalArgs(C.Structure):
    """fsb_eval_args (include/fastsum_b200.h)."""
    _fields_ = [("method", _I), ("kid", _I), ("alpha", _D), ("dfloor", _D), ("precision", _I),
                ("beta", _D), ("n_samples", _I64), ("rr_mode", _I), ("seed", C.c_uint64),
                ("query_offset", _I64), ("smooth", _I), ("query_order", _I),
                ("src_pts", _P), ("src_ms", _P), ("m", _I64), ("c", _I),
                ("rng_group_log2", _I), ("bh_warp_vote", _I), ("path_variant", _I)]


METHOD_CODES = {"brute_force": 0, "barnes_hut": 1, "telescoping_exhaustive": 2, "stochastic": 3}

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "fsb_abi_version": [],
    "fsb_last_error": [],
    "fsb_brute_force_batch": [_I, _D, _D, _I, _P, _P, _I64, _I, _P, _I64, _P, _P],
    "fsb_brute_force_f32acc64": [_I, _D, _D, _P, _P, _I64, _I, _P, _I64, _P, _P],
    "fsb_build_tree": [_P, _P, _P, _I64, _I, _I, _I, C.POINTER(_P), _P],
    "fsb_tree_from_core_arrays": [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I,
                                  C.POINTER(_P), _P],
    "fsb_tree_info": [_P, C.POINTER(_I64)],
    "fsb_tree_export": [_P, C.POINTER(_P), _P],
    "fsb_tree_free": [_P],
    "fsb_barnes_hut_batch": [_P, _I, _D, _D, _I, _P, _I64, _P, _D, _P, _P, _P],
    "fsb_barnes_hut_vote_batch": [_P, _I, _D, _D, _I, _P, _I64, _P, _D, _P, _P, _P],
    "fsb_stochastic_batch": [_P, _I, _D, _D, _I, _P, _I64, _P, _I64, _I, C.c_uint64, _I64, _P,
                             _P, _P, _P, _P],
    "fsb_stochastic_batch_ex": [_P, _I, _D, _D, _I, _P, _I64, _P, _I64, _I, C.c_uint64, _I64,
                                _I, _I, _P, _P, _P, _P, _P],
    "fsb_stochastic_moments_batch": [_P, _I, _D, _D, _P, _I64, _I64, _I, C.c_uint64, _P, _P, _P],
    "fsb_telescoping_batch": [_P, _I, _D, _D, _I, _P, _I64, _P, _P, _P],
    "fsb_query_order": [_P, _I64, _P, _P],
    "fsb_shuffle_order": [_I64, C.c_uint64, _I64, _P, _P],
    "fsb_post_transform": [_P, _I, _I64, _I, _D, _P, _P, _P, _P],
    "fsb_evaluate_field_host": [_P, C.POINTER(EvalArgs), _P, _I64, _P, _P, _P, _P, _P, _P, _I,
                                _P],
    "fsb_error_stats": [_P, _P, _P, _P, _I64, _P, C.POINTER(_I64), _P],
    "fsb_sample_mesh_surface": [_P, _I64, _P, _P, _I64, _P, _D, _D, _P, _P, _P, _P],
    "fsb_make_queries": [_I, _I64, _P, _P, _P, _I64, _I64, _P, _P, _P, _P],
    "fsb_write_field_csv": [C.c_char_p, _I64, _P, _P, _P],
    "fsb_write_points_file": [C.c_char_p, _I64, _I, _P, _P],
    "fsb_selftest_fp64": [_I64, C.c_uint64, _P],
    "fsb_selftest_bh_far": [_I64, C.c_uint64, _P],
    "fsb_micro_peaks": [_P, _P],
    "fsb_gate": [_P, C.c_int64, _P],
}
_RESTYPES = {"fsb_last_error": C.c_char_p}


class FastsumError(RuntimeError):
    pass


def load(build_if_missing: bool = True):
    """Load (and if needed build) the CUDA library; does not need a GPU."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if not build_if_missing:
                raise FastsumError(f"CUDA library missing: {LIB_PATH} (run __graft_entry__.build())")
            from . import _build
            _build.build()
        lib = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = lib
        return lib


def lib():
    """The library, for compute calls: requires a CUDA device (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise FastsumError("paper_2506_02219_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    return load()


def check(rc: int) -> None:
    if rc != 0:
        msg = load().fsb_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(msg)
        raise FastsumError(msg)
