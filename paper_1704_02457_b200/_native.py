"""ctypes binding of the C ABI in include/pb_b200.h (libpb_b200.so).

This is the Python side of the drop-in boundary: it plays the role the
reference's backend selector plays (_backend/__init__.py:12-44), except
that there is exactly one backend.  There is no CPU fallback: if the
native library cannot be loaded, every call raises.
"""
from __future__ import annotations

import ctypes
import os

from . import _build

_lib = None
_load_error = None


class DmatBatch(ctypes.Structure):
    """Mirror of ``pb_dmat_batch`` (include/pb_b200.h)."""

    _fields_ = [
        ("pA", ctypes.c_void_p),
        ("dA", ctypes.c_void_p),
        ("m", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("cn", ctypes.c_int32),
        ("batch", ctypes.c_int32),
        ("stride", ctypes.c_int64),
        ("dA_stride", ctypes.c_int64),
    ]


ABI_VERSION = 2
P = ctypes.POINTER(DmatBatch)
_i, _d, _v, _l = ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64

# name -> (restype, argtypes); the exact exported surface of pb_b200.h
SIGNATURES = {
    "pb_version": (_i, []),
    "pb_last_error": (ctypes.c_char_p, []),
    "pb_launch_count": (_l, [_i]),
    "pb_dgemm_nt": (_i, [_i, _i, _i, _d, P, _i, _i, P, _i, _i, _d, P, _i, _i, P, _i, _i, _v]),
    "pb_dsyrk_ln": (_i, [_i, _i, _d, P, _i, _i, P, _i, _i, _d, P, _i, _i, P, _i, _i, _v]),
    "pb_dtrsm_rltn": (_i, [_i, _i, _d, P, _i, _i, _i, P, _i, _i, P, _i, _i, _v, _v]),
    "pb_dpotrf_l": (_i, [_i, _i, P, _i, _i, P, _i, _i, _v, _v, _l, _v]),
    "pb_dpotrf_l_worksize": (_l, [_i, _i, P, _i, _i, P, _i, _i]),
    "pb_dpack_cm": (_i, [_i, _i, _v, _l, _l, P, _i, _i, _v]),
    "pb_dunpack_cm": (_i, [_i, _i, P, _i, _i, _v, _l, _l, _v]),
    "pb_dpack": (_i, [_i, _i, _v, _l, _l, _l, P, _i, _i, _v]),
    "pb_dunpack": (_i, [_i, _i, P, _i, _i, _v, _l, _l, _l, _v]),
    "pb_dgecp": (_i, [_i, _i, P, _i, _i, P, _i, _i, _v]),
    "pb_dgemm_nn": (_i, [_i, _i, _i, _d, P, _i, _i, P, _i, _i, _d, P, _i, _i, P, _i, _i, _v]),
    "pb_dtrmm_rlnn": (_i, [_i, _i, _d, P, _i, _i, P, _i, _i, P, _i, _i, _v, _l, _v]),
    "pb_dtrmm_rlnn_worksize": (_l, [_i, _i, P, _i, _i, P, _i, _i, P, _i, _i]),
    "pb_dsyrk_potrf_ln": (_i, [_i, _i, _i, P, _i, _i, P, _i, _i, P, _i, _i, P, _i, _i, _v, _v, _l, _v]),
    "pb_dsyrk_potrf_ln_worksize": (_l, [_i, _i, _i, P, _i, _i, P, _i, _i, P, _i, _i, P, _i, _i]),
    "pb_driccati_chain": (_i, [_i, _i, _i, P, P, P, P, _v, _v]),
    "pb_dgetrf": (_i, [_i, _i, P, _i, _i, P, _i, _i, _i, _v, _l, _v, _v]),
}


def lib_path():
    return _build.LIB_PATH


def load():
    """Load (building first if needed and possible) the native library."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    try:
        if not _build.up_to_date():
            if _build.nvcc_path() is not None:
                _build.build()
            elif not os.path.exists(_build.LIB_PATH):
                raise RuntimeError("libpb_b200.so is missing and nvcc is unavailable")
        lib = ctypes.CDLL(_build.LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.pb_version() != ABI_VERSION:
            raise RuntimeError("libpb_b200.so ABI version mismatch")
    except Exception as exc:  # no fallback: remember and re-raise loudly
        _load_error = exc
        raise RuntimeError(f"panel-major CUDA engine unavailable: {exc}") from exc
    _lib = lib
    return lib


def call(name, *args):
    """Invoke an ABI function; non-zero status raises with pb_last_error()."""
    lib = load()
    st = getattr(lib, name)(*args)
    if st != 0:
        msg = lib.pb_last_error().decode(errors="replace")
        raise RuntimeError(f"{name} failed with status {st}: {msg}")
    return st


def worksize(name, *args):
    """Bytes of caller-owned workspace ``name`` needs for these arguments
    (its ``<name>_worksize`` query); raises like :func:`call` on a bad argument."""
    lib = load()
    v = getattr(lib, name + "_worksize")(*args)
    if v < 0:
        msg = lib.pb_last_error().decode(errors="replace")
        raise RuntimeError(f"{name}_worksize failed with status {v}: {msg}")
    return int(v)


def workspace(nbytes, device):
    """A device workspace of ``nbytes`` from PyTorch's caching allocator on
    the current stream (the reference's L3 allocates its scratch the same
    way, level3.py:59, 236, 338): (tensor-or-None, pointer, bytes)."""
    if nbytes <= 0:
        return None, ctypes.c_void_p(0), 0
    import torch
    t = torch.empty((nbytes + 255) // 8 + 32, dtype=torch.float64, device=device)
    base = t.data_ptr()
    shift = (-base) % 256
    return t, ctypes.c_void_p(base + shift), nbytes


def launch_count(reset=False):
    return int(load().pb_launch_count(1 if reset else 0))
