"""Device-side operations on torch CUDA tensors, all computed by the sm_100a
kernels behind the C ABI (include/tsnmf_b200.h).

PyTorch is plumbing here: it owns device memory, the current CUDA stream and
(in ``sharded``) the NCCL process group.  Every arithmetic step of the
reduction runs in ``libtsnmf_b200.so``; a missing library or a missing GPU
raises instead of falling back to a CPU path.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native
from .errors import TsnmfError, UsageError

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_device(device=None):
    """The CUDA device to run on; raises if there is none (no CPU fallback)."""
    t = torch()
    _native.load()
    if not t.cuda.is_available():
        raise TsnmfError("no CUDA device: the B200 reduction path has no CPU fallback", stage="device")
    if device is None:
        return t.device("cuda", t.cuda.current_device())
    device = t.device(device)
    if device.type != "cuda":
        raise UsageError(f"expected a CUDA device, got {device}")
    return device


def stream_ptr(device=None) -> int:
    return torch().cuda.current_stream(device).cuda_stream


class _WorkspaceCache:
    """Grow-only scratch buffer per (device, stream).  Freed buffers are reused
    by torch's caching allocator in stream order, so growing is safe."""

    def __init__(self):
        self._lock = threading.Lock()
        self._bufs: dict = {}

    def get(self, nbytes: int, device) -> tuple[int, int]:
        t = torch()
        key = (device.index, t.cuda.current_stream(device).cuda_stream)
        with self._lock:
            buf = self._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = t.empty(max(int(nbytes), 1 << 20), dtype=t.uint8, device=device)
                self._bufs[key] = buf
            return buf.data_ptr(), buf.numel()

    def clear(self):
        with self._lock:
            self._bufs.clear()


workspaces = _WorkspaceCache()


def _workspace(op: int, m: int, n: int, k: int, device) -> tuple[int, int]:
    need = _native.load().tsnmf_workspace_bytes(op, int(m), int(n), int(k))
    if need == 0:
        raise UsageError(f"unsupported problem size for op {op}: m={m}, n={n}, k={k} "
                         f"(max columns {max_cols()})", stage="device")
    return workspaces.get(need, device)


def max_cols() -> int:
    return int(_native.load().tsnmf_max_cols())


def as_device_matrix(data, device=None):
    """2-D float64 CUDA tensor with unit column stride (rows may be strided)."""
    t = torch()
    dev = require_device(device if device is not None else (data.device if isinstance(data, t.Tensor)
                                                            and data.is_cuda else None))
    if isinstance(data, t.Tensor):
        x = data
    else:
        arr = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
        x = t.from_numpy(arr if arr.flags.writeable else arr.copy())
    if x.dim() != 2:
        raise UsageError(f"chunk must be a 2-D matrix, got shape {tuple(x.shape)}")
    if x.dtype != t.float64:
        x = x.to(t.float64)
    if not x.is_cuda or x.device != dev:
        x = x.to(dev, non_blocking=True)
    if x.shape[0] > 0 and (x.stride(1) != 1 or x.stride(0) < x.shape[1]):
        x = x.contiguous()
    return x


def _ld(x) -> int:
    return int(x.stride(0)) if x.shape[0] > 1 else int(x.shape[1])


# ---------------------------------------------------------------------------
# reductions


def tsqr(x, *, stats: bool = True):
    """(R, l1, sumsq) of a device row block; R is n x n, sign-fixed upper
    triangular (reference tsqr.py:129-141 + tsqr.py:190-192)."""
    t = torch()
    x = as_device_matrix(x)
    m, n = int(x.shape[0]), int(x.shape[1])
    if m < 1:
        raise UsageError(f"chunk must have at least one row, got shape {(m, n)}")
    dev = x.device
    r = t.empty((n, n), dtype=t.float64, device=dev)
    l1 = t.empty(n, dtype=t.float64, device=dev) if stats else None
    sq = t.empty(n, dtype=t.float64, device=dev) if stats else None
    ws, wsb = _workspace(_native.OP_TSQR, m, n, 0, dev)
    _native.call("tsnmf_tsqr", x.data_ptr(), m, n, _ld(x), r.data_ptr(), n,
                 l1.data_ptr() if stats else None, sq.data_ptr() if stats else None, ws, wsb,
                 stream_ptr(dev), device=dev, stage="tsqr")
    return r, l1, sq


def combine_factors(rs):
    """R of the vertical stack of factors rs (count x n x n device tensor),
    combined in TreeReducer order (reference tsqr.py:144-153, 201-234)."""
    t = torch()
    rs = rs.contiguous()
    count, n = int(rs.shape[0]), int(rs.shape[1])
    dev = rs.device
    r = t.empty((n, n), dtype=t.float64, device=dev)
    ws, wsb = _workspace(_native.OP_COMBINE, count, n, 0, dev)
    _native.call("tsnmf_r_combine", rs.data_ptr(), count, n, r.data_ptr(), n, ws, wsb, stream_ptr(dev), device=dev,
                 stage="combine")
    return r


def gram(x, *, stats: bool = True):
    """(X^T X, l1, sumsq) of a device row block."""
    t = torch()
    x = as_device_matrix(x)
    m, n = int(x.shape[0]), int(x.shape[1])
    dev = x.device
    g = t.empty((n, n), dtype=t.float64, device=dev)
    l1 = t.empty(n, dtype=t.float64, device=dev) if stats else None
    sq = t.empty(n, dtype=t.float64, device=dev) if stats else None
    ws, wsb = _workspace(_native.OP_GRAM, m, n, 0, dev)
    _native.call("tsnmf_gram", x.data_ptr(), m, n, _ld(x), g.data_ptr(), n,
                 l1.data_ptr() if stats else None, sq.data_ptr() if stats else None, ws, wsb,
                 stream_ptr(dev), device=dev, stage="gram")
    return g, l1, sq


def sketch(x, row_offset: int, seed: int, k: int, g=None):
    """G^T X (k x n) with G[i, t] = normal #((row_offset+i)*k + t) of the
    sketch stream of ``seed`` (reference sketch.py:62-73, rng.py:48-55), or
    with an explicit device G (m x k)."""
    t = torch()
    x = as_device_matrix(x)
    m, n = int(x.shape[0]), int(x.shape[1])
    dev = x.device
    s = t.empty((k, n), dtype=t.float64, device=dev)
    gp, ldg = None, 0
    if g is not None:
        g = as_device_matrix(g, dev)
        if tuple(g.shape) != (m, k):
            raise UsageError(f"explicit G must be {(m, k)}, got {tuple(g.shape)}")
        gp, ldg = g.data_ptr(), _ld(g) if m > 1 else k
    ws, wsb = _workspace(_native.OP_SKETCH, m, n, k, dev)
    _native.call("tsnmf_sketch", x.data_ptr(), m, n, _ld(x), int(row_offset), int(seed) & ((1 << 64) - 1), int(k),
                 gp, ldg, s.data_ptr(), n, ws, wsb, stream_ptr(dev), device=dev, stage="sketch")
    return s


def column_stats(x):
    t = torch()
    x = as_device_matrix(x)
    m, n = int(x.shape[0]), int(x.shape[1])
    dev = x.device
    l1 = t.empty(n, dtype=t.float64, device=dev)
    sq = t.empty(n, dtype=t.float64, device=dev)
    ws, wsb = _workspace(_native.OP_STATS, m, n, 0, dev)
    _native.call("tsnmf_column_stats", x.data_ptr(), m, n, _ld(x), l1.data_ptr(), sq.data_ptr(), ws, wsb,
                 stream_ptr(dev), device=dev, stage="stats")
    return l1, sq


def first_nonfinite(x) -> int:
    """Linear (row-major) index of the first Inf/NaN of a contiguous device array, -1 if none
    (reference matio.py:81-87 _check_finite, on the device)."""
    t = torch()
    if not (isinstance(x, t.Tensor) and x.is_cuda and x.dtype == t.float64 and x.is_contiguous()):
        raise UsageError("first_nonfinite needs a contiguous CUDA float64 tensor")
    dev = x.device
    out = t.empty(1, dtype=t.int64, device=dev)
    _native.call("tsnmf_first_nonfinite", x.data_ptr(), int(x.numel()), out.data_ptr(), stream_ptr(dev), device=dev,
                 stage="read")
    return int(out.item())


# ---------------------------------------------------------------------------
# selection / coefficients


def nnls(a, b, *, tol: float = 1e-8, max_iter: int = 10_000):
    """Batched NNLS on the device: Y[:, j] = argmin ||a y - b[:, j]||, y >= 0 (reference nnls.py:47-126).
    a: n x t design, b: n x ncols targets (host or device).  Returns (Y t x ncols, status ncols) device
    tensors; status 0 ok, 3 numerical, 5 iteration limit."""
    t = torch()
    a = as_device_matrix(a)
    dev = a.device
    b = as_device_matrix(b, dev)
    n, q = int(a.shape[0]), int(a.shape[1])
    if int(b.shape[0]) != n:
        raise UsageError(f"incompatible shapes {tuple(a.shape)} and {tuple(b.shape)}", stage="nnls")
    ncols = int(b.shape[1])
    y = t.empty((q, ncols), dtype=t.float64, device=dev)
    status = t.empty(ncols, dtype=t.int32, device=dev)
    ws, wsb = _workspace(_native.OP_NNLS, 1, q, 0, dev)
    _native.call("tsnmf_nnls", a.data_ptr(), n, q, _ld(a), b.data_ptr(), _ld(b), ncols, float(tol), int(max_iter),
                 y.data_ptr(), ncols, status.data_ptr(), ws, wsb, stream_ptr(dev), device=dev, stage="nnls")
    return y, status


def nnls_max_cols() -> int:
    return int(_native.load().tsnmf_nnls_max_cols())


def xray_scores(m, resid, colnorm):
    """score[j] = ||resid^T m[:, j]|| / colnorm[j] (-inf where colnorm <= 0) (reference select.py:131-135)."""
    t = torch()
    n = int(m.shape[0])
    score = t.empty(n, dtype=t.float64, device=m.device)
    _native.call("tsnmf_xray_scores", m.data_ptr(), n, _ld(m), resid.data_ptr(), _ld(resid), colnorm.data_ptr(),
                 score.data_ptr(), stream_ptr(m.device), device=m.device, stage="xray")
    return score


def xray_residual(m, a, coef, out):
    """out = m - a @ coef (reference select.py:138-140)."""
    n, q = int(m.shape[0]), int(a.shape[1])
    _native.call("tsnmf_xray_residual", m.data_ptr(), n, _ld(m), a.data_ptr(), q, _ld(a), coef.data_ptr(),
                 _ld(coef), out.data_ptr(), _ld(out), stream_ptr(m.device), device=m.device, stage="xray")
    return out


def scale_columns(a, norms):
    """a D^-1 with D = diag(norms) (reference tsqr.py:163-177, sketch.py:87-100), on the device."""
    t = torch()
    a = as_device_matrix(a)
    norms = as_device_matrix(norms.reshape(1, -1) if hasattr(norms, "reshape") else np.asarray(norms)[None, :],
                             a.device).reshape(-1)
    out = t.empty(a.shape, dtype=t.float64, device=a.device)
    _native.call("tsnmf_scale_columns", a.data_ptr(), int(a.shape[0]), int(a.shape[1]), _ld(a), norms.data_ptr(),
                 out.data_ptr(), int(out.shape[1]), stream_ptr(a.device), device=a.device, stage="scale")
    return out


def gp_select(sk, r: int):
    """GP selection order on the device (reference select.py:159-178): (indices tensor, count)."""
    t = torch()
    sk = as_device_matrix(sk)
    out = t.empty(int(r), dtype=t.int32, device=sk.device)
    cnt = t.empty(1, dtype=t.int32, device=sk.device)
    _native.call("tsnmf_gp_select", sk.data_ptr(), int(sk.shape[0]), int(sk.shape[1]), _ld(sk), int(r),
                 out.data_ptr(), cnt.data_ptr(), stream_ptr(sk.device), device=sk.device, stage="select-gp")
    return out, cnt


def svd_reduced(r):
    """Singular values and right singular vectors of the n x n factor on the device (cuSOLVER via torch: a
    library SVD, like cuBLAS for a plain GEMM).  Row signs of V^T are LAPACK's choice on either side; every
    consumer of the reduced matrix (SPA, XRAY, NNLS) is invariant under them."""
    t = torch()
    r = as_device_matrix(r)
    _, s, vt = t.linalg.svd(r, full_matrices=False)
    return s, vt


# ---------------------------------------------------------------------------
# counter RNG blocks


def uniform_block(stream: int, start: int, count: int, device=None):
    t = torch()
    dev = require_device(device)
    out = t.empty(int(count), dtype=t.float64, device=dev)
    _native.call("tsnmf_uniform_block", int(stream) & ((1 << 64) - 1), int(start) & ((1 << 64) - 1), int(count),
                 out.data_ptr(), stream_ptr(dev), device=dev, stage="rng")
    return out


def normal_block(stream: int, start: int, count: int, device=None):
    t = torch()
    dev = require_device(device)
    out = t.empty(int(count), dtype=t.float64, device=dev)
    _native.call("tsnmf_normal_block", int(stream) & ((1 << 64) - 1), int(start) & ((1 << 64) - 1), int(count),
                 out.data_ptr(), stream_ptr(dev), device=dev, stage="rng")
    return out


def gaussian_rows(seed: int, row_offset: int, rows: int, k: int, device=None):
    t = torch()
    dev = require_device(device)
    out = t.empty((int(rows), int(k)), dtype=t.float64, device=dev)
    _native.call("tsnmf_gaussian_rows", int(seed) & ((1 << 64) - 1), int(row_offset), int(rows), int(k),
                 out.data_ptr(), stream_ptr(dev), device=dev, stage="rng")
    return out


def derive_stream(seed: int, tag: int) -> int:
    return int(_native.load().tsnmf_derive_stream(int(seed) & ((1 << 64) - 1), int(tag) & ((1 << 64) - 1)))


def tsqr_plan(n: int, m: int) -> dict:
    vals = [ctypes.c_int32() for _ in range(4)]
    _native.check(_native.load().tsnmf_tsqr_plan(int(n), int(m), *[ctypes.byref(v) for v in vals]))
    return dict(zip(("panel", "block_rows", "ctas_per_sm", "leaves"), (v.value for v in vals)))
