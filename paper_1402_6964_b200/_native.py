"""ctypes binding of the C ABI in include/tsnmf_b200.h (libtsnmf_b200.so, built in-tree).

There is no fallback: if the shared library is missing or no CUDA device is
present, every device entry point raises.  Status codes map onto the
reference's exception classes (reference pkg/src/tsnmf/errors.py:16-31).
"""

from __future__ import annotations

import ctypes
import os

from .errors import DataError, NumericalError, TsnmfError, UsageError

LIB_NAME = "libtsnmf_b200.so"
LIB_PATH = os.environ.get("TSNMF_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
ABI_VERSION = 1

OP_TSQR, OP_COMBINE, OP_GRAM, OP_SKETCH, OP_STATS, OP_NNLS = 1, 2, 3, 4, 5, 6

_u64, _i64, _i32, _vp, _sz, _dbl = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                    ctypes.c_size_t, ctypes.c_double)

# name -> (restype, argtypes); mirrors include/tsnmf_b200.h one-for-one
SIGNATURES = {
    "tsnmf_abi_version": (ctypes.c_int, []),
    "tsnmf_last_error": (ctypes.c_char_p, []),
    "tsnmf_max_cols": (ctypes.c_int, []),
    "tsnmf_workspace_bytes": (_sz, [ctypes.c_int, _i64, _i32, _i32]),
    "tsnmf_derive_stream": (_u64, [_u64, _u64]),
    "tsnmf_uniform_block": (ctypes.c_int, [_u64, _u64, _i64, _vp, _vp]),
    "tsnmf_normal_block": (ctypes.c_int, [_u64, _u64, _i64, _vp, _vp]),
    "tsnmf_gaussian_rows": (ctypes.c_int, [_u64, _i64, _i64, _i32, _vp, _vp]),
    "tsnmf_tsqr": (ctypes.c_int, [_vp, _i64, _i32, _i64, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "tsnmf_r_combine": (ctypes.c_int, [_vp, _i32, _i32, _vp, _i64, _vp, _sz, _vp]),
    "tsnmf_gram": (ctypes.c_int, [_vp, _i64, _i32, _i64, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "tsnmf_sketch": (ctypes.c_int, [_vp, _i64, _i32, _i64, _i64, _u64, _i32, _vp, _i64, _vp, _i64, _vp, _sz, _vp]),
    "tsnmf_column_stats": (ctypes.c_int, [_vp, _i64, _i32, _i64, _vp, _vp, _vp, _sz, _vp]),
    "tsnmf_first_nonfinite": (ctypes.c_int, [_vp, _i64, _vp, _vp]),
    "tsnmf_scale_columns": (ctypes.c_int, [_vp, _i32, _i32, _i64, _vp, _vp, _i64, _vp]),
    "tsnmf_gp_select": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _vp, _vp, _vp]),
    "tsnmf_generate": (ctypes.c_int, [_vp, _i64, _i64, _i64, _i32, _i32, _vp, _i32, _vp, _i64, _dbl, _u64, _vp]),
    "tsnmf_nnls": (ctypes.c_int, [_vp, _i64, _i32, _i64, _vp, _i64, _i32, _dbl, _i32, _vp, _i64, _vp, _vp, _sz, _vp]),
    "tsnmf_nnls_max_cols": (ctypes.c_int, []),
    "tsnmf_xray_scores": (ctypes.c_int, [_vp, _i32, _i64, _vp, _i64, _vp, _vp, _vp]),
    "tsnmf_xray_residual": (ctypes.c_int, [_vp, _i32, _i64, _vp, _i32, _i64, _vp, _i64, _vp, _i64, _vp]),
    "tsnmf_launch_count": (ctypes.c_longlong, []),
    "tsnmf_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "tsnmf_profile_read": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_longlong)]),
    "tsnmf_tsqr_plan": (ctypes.c_int, [_i32, _i64, ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                                       ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
}

_lib = None


class NativeLibraryMissing(TsnmfError):
    """The CUDA extension is not built; there is no CPU fallback."""


def load(path: str = LIB_PATH):
    """Load (once) and return the shared library with typed entry points."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryMissing(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)", stage="load")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.tsnmf_abi_version() != ABI_VERSION:
        raise NativeLibraryMissing(f"ABI mismatch: library {lib.tsnmf_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


_ERRORS = {1: UsageError, 2: DataError, 3: NumericalError}


def check(status: int, stage: str = "device") -> None:
    """Raise the reference-compatible exception for a non-zero status."""
    if status == 0:
        return
    msg = load().tsnmf_last_error().decode(errors="replace")
    cls = _ERRORS.get(status)
    if cls is None:
        raise TsnmfError(f"CUDA failure: {msg}", stage=stage)
    raise cls(msg, stage=stage)


def call(name: str, *args, stage: str = "device", device=None) -> None:
    """Call one C-ABI entry point.  With ``device`` the call runs with that CUDA device current: the
    library launches on the stream it is given but sets per-device kernel attributes and queries the
    SM count of the *current* device, so the two must agree."""
    fn = getattr(load(), name)
    if device is None:
        check(fn(*args), stage=stage)
        return
    import torch

    with torch.cuda.device(device):
        check(fn(*args), stage=stage)
