"""The B200 backend as the reference package itself loads it.

The reference ``tsnmf`` (pure Python + one Cython RNG) has exactly one plugin point: the block-kernel
backend chosen by ``TSNMF_BACKEND`` in reference ``kernels.py:13-31``, whose module contract is
``BACKEND``, ``uniform_block(stream, start, count)`` and ``normal_block(stream, start, count)`` returning
callee-allocated float64 arrays (reference ``_kernels.pyx:35-69``).  This module satisfies that contract
with the device counter RNG (``tsnmf_uniform_block`` / ``tsnmf_normal_block`` in libtsnmf_b200.so), and
``install`` routes the reference's one-pass reduction onto the device so that everything downstream of it —
``pipeline.run_factorize`` / ``run_sweep``, the artifact cache, selection, NNLS, the CLI — runs UNCHANGED
on the reference's own code:

    reference symbol (file:line)                  rebound to
    kernels.uniform_block / normal_block :27-28   this module's block kernels (``get_backend()`` = "b200")
    tsqr.stream_pass              tsqr.py:276     device pass (factor.stream_pass): TSQR leaf + tree
    tsqr.factor_chunk             tsqr.py:129     device TSQR of one chunk
    tsqr.combine                  tsqr.py:144     device combine of a stacked pair
    sketch.sketch_chunk           sketch.py:62    device GX (G generated in the kernel, or the hook's G)
    nnls.solve_columns (optional) nnls.py:106     batched device Lawson-Hanson (``select=True``)

Results come back as the reference's own types (``tsqr.TriangularFactor``, ``tsqr.ColumnStats``,
``sketch.SketchResult``, ``tsqr.StreamResult``) and errors as the reference's own exception classes with
the same message and stage, so the reference's ``_stage`` tagging and CLI exit codes still apply.
The package-level re-exports (``tsnmf.stream_pass`` ...) are rebound too.

Two ways in:
  * unmodified reference:  ``import tsnmf; refbackend.install(tsnmf)``;
  * maintainer patch (``KERNELS_PATCH`` / ``INIT_PATCH`` below, 6 lines): ``TSNMF_BACKEND=b200`` selects this
    module in ``kernels.py`` and ``tsnmf/__init__`` calls ``install`` on import.
There is no CPU fallback: without a GPU or the library every call raises.
"""

from __future__ import annotations

import sys

import numpy as np

from . import device as dv
from . import errors as own_errors

BACKEND = "b200"

_MASK = (1 << 64) - 1


# ---------------------------------------------------------------------------
# block-kernel backend contract (reference _kernels.pyx:35-69; values: uniforms bit-exact, normals within
# the reference's own backend tolerance, reference tests/test_kernels.py:40-49)


def uniform_block(stream, start, count) -> np.ndarray:
    """Uniform [0, 1) doubles at counters start .. start+count-1 of ``stream`` (callee-allocated)."""
    count = int(count)
    if count <= 0:
        return np.empty(0, dtype=np.float64)
    return dv.uniform_block(int(stream) & _MASK, int(start) & _MASK, count).cpu().numpy()


def normal_block(stream, start, count) -> np.ndarray:
    """Standard normals at indices start .. start+count-1 of ``stream`` (callee-allocated)."""
    count = int(count)
    if count <= 0:
        return np.empty(0, dtype=np.float64)
    return dv.normal_block(int(stream) & _MASK, int(start) & _MASK, count).cpu().numpy()


# ---------------------------------------------------------------------------
# the maintainer patch (applied to a scratch copy by tests/test_refbackend.py; shown in INTEGRATION.md)

KERNELS_ANCHOR = 'if _choice == "python":'
KERNELS_PATCH = (
    'if _choice == "b200":\n'
    '    from paper_1402_6964_b200 import refbackend as _impl  # type: ignore[no-redef]\n'
    'elif _choice == "python":'
)
INIT_PATCH = (
    "\n# B200 backend: route the one-pass reduction onto the GPU (paper_1402_6964_b200, INTEGRATION.md)\n"
    "from . import kernels as _kernels\n"
    "if _kernels._choice == \"b200\":\n"
    "    from paper_1402_6964_b200 import refbackend as _b200\n"
    "    _b200.install(__import__(__name__))\n"
)


def patch_reference_tree(pkg_dir) -> None:
    """Apply the 6-line maintainer patch to a writable copy of the reference package directory
    (``.../tsnmf``): the ``b200`` choice in ``kernels.py`` and the ``install`` hook in ``__init__.py``."""
    from pathlib import Path

    pkg_dir = Path(pkg_dir)
    kp = pkg_dir / "kernels.py"
    src = kp.read_text()
    if "refbackend" not in src:
        if KERNELS_ANCHOR not in src:
            raise own_errors.UsageError(f"{kp}: backend selection anchor not found")
        kp.write_text(src.replace(KERNELS_ANCHOR, KERNELS_PATCH, 1))
    ip = pkg_dir / "__init__.py"
    src = ip.read_text()
    if "refbackend" not in src:
        ip.write_text(src + INIT_PATCH)


# ---------------------------------------------------------------------------
# routing the reference's hot path


def _translate(ref_errors):
    """Context manager re-raising this package's errors as the reference's classes (same name, message,
    stage; the original is chained)."""
    from contextlib import contextmanager

    @contextmanager
    def cm():
        try:
            yield
        except own_errors.TsnmfError as exc:
            if isinstance(exc, ref_errors.TsnmfError):
                raise
            cls = getattr(ref_errors, type(exc).__name__, None)
            if cls is None:
                for base in type(exc).__mro__:
                    cls = getattr(ref_errors, base.__name__, None)
                    if cls is not None:
                        break
            raise cls(str(exc), stage=exc.stage) from exc

    return cm


def _ref_nnls_iteration(ref, exc):
    """A device iteration-cap failure as the reference raises it: NumericalError("column i: ...") caused by
    the reference's NnlsIterationError carrying best_y / kkt_violation (nnls.py:96-103,117-121)."""
    inner = exc.__cause__ if exc.__cause__ is not None else exc
    best_y = getattr(inner, "best_y", None)
    kkt = getattr(inner, "kkt_violation", None)
    cause = ref.nnls.NnlsIterationError(str(inner), best_y=best_y, kkt_violation=kkt) if best_y is not None else None
    return ref.errors.NumericalError(str(exc)), cause


def install(ref=None, *, select: bool = False):
    """Rebind the reference package's hot-path entry points onto the device (see the module table).

    ``ref`` is the imported reference package (default: ``sys.modules["tsnmf"]``).  With ``select=True``
    the reference's per-column NNLS (``nnls.solve_columns``, used by ``compute_h``, XRAY's refits and the
    sweep) runs as one batched device Lawson-Hanson.  Returns ``ref``."""
    if ref is None:
        ref = sys.modules["tsnmf"]
    from . import factor as own_factor
    from . import nonneg as own_nonneg
    from . import projection as own_proj

    kernels, tsqr, sketch_mod, nnls = ref.kernels, ref.tsqr, ref.sketch, ref.nnls
    xlate = _translate(ref.errors)
    dv.require_device()  # fail loudly now, not on the first chunk

    def stream_pass(chunks, *, sketch_rows=None, seed=0, combine_order="tree", threads=1):
        with xlate():
            res = own_factor.stream_pass(chunks, sketch_rows=sketch_rows, seed=seed,
                                         combine_order=combine_order, threads=threads)
        stats = tsqr.ColumnStats(l1=np.array(res.stats.l1), l2=np.array(res.stats.l2))
        sk = None if res.sketch is None else sketch_mod.SketchResult(entries=np.array(res.sketch.entries),
                                                                      seed=res.sketch.seed)
        return tsqr.StreamResult(factor=tsqr.TriangularFactor(entries=np.array(res.factor.entries)), stats=stats,
                                 sketch=sk, rows=res.rows, chunks=res.chunks, tree_depth=res.tree_depth)

    def factor_chunk(chunk):
        with xlate():
            r = own_factor.factor_chunk(chunk)
        return tsqr.TriangularFactor(entries=np.array(r.entries))

    def combine(r1, r2):
        with xlate():
            r = own_factor.combine(own_factor.TriangularFactor(entries=np.array(r1.entries)),
                                   own_factor.TriangularFactor(entries=np.array(r2.entries)))
        return tsqr.TriangularFactor(entries=np.array(r.entries))

    def sketch_chunk(chunk, k, seed, *, gaussian_rows_fn=None):
        with xlate():
            s = own_proj.sketch_chunk(chunk, k, seed, gaussian_rows_fn=gaussian_rows_fn)
        return sketch_mod.SketchResult(entries=np.array(s.entries), seed=seed)

    def solve_columns(design, targets, *, tol=1e-8, threads=1):
        try:
            with xlate():
                return own_nonneg.solve_columns(design, targets, tol=tol, threads=threads, device=True)
        except ref.errors.NumericalError as exc:
            if isinstance(exc.__cause__, own_errors.NumericalError) and exc.__cause__.__cause__ is not None:
                out, cause = _ref_nnls_iteration(ref, exc.__cause__)
                raise out from cause
            raise

    stream_pass.__doc__ = own_factor.stream_pass.__doc__
    kernels._impl = sys.modules[__name__]
    kernels.uniform_block = uniform_block
    kernels.normal_block = normal_block
    tsqr.stream_pass = stream_pass
    tsqr.factor_chunk = factor_chunk
    tsqr.combine = combine
    sketch_mod.sketch_chunk = sketch_chunk
    for name, fn in (("stream_pass", stream_pass), ("factor_chunk", factor_chunk), ("combine", combine),
                     ("sketch_chunk", sketch_chunk)):
        setattr(ref, name, fn)
    if select:
        nnls.solve_columns = solve_columns
    ref.__b200_installed__ = True
    return ref


__all__ = ["BACKEND", "INIT_PATCH", "KERNELS_PATCH", "install", "normal_block", "patch_reference_tree",
           "uniform_block"]
