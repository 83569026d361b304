"""Single-pass TSQR / Gram reduction with fused column statistics — drop-in
for reference pkg/src/tsnmf/tsqr.py (same names, signatures, result types and
error behaviour), computed on the B200.

Semantics kept from the reference:
  * ``TriangularFactor`` / ``ColumnStats`` / ``ReducedSVD`` / ``StreamResult``
    validation and read-only arrays (tsqr.py:27-110, 237-244);
  * ``combine_order``: "tree" (binary-counter tree over the chunk index,
    deterministic), "sequential" (left fold), "first-come" (tree with
    threads == 1, as in the reference; a left fold in arrival order with
    threads > 1) (tsqr.py:24, 294-333);
  * errors: empty stream -> DataError, m < n -> DataError("not tall-and-skinny"),
    bad order / threads -> UsageError (tsqr.py:294-297, 335-341).

What changes: every chunk is reduced by ``libtsnmf_b200.so`` (device.py).
Device-resident chunks (torch CUDA float64) are reduced in place; host chunks
(numpy) are gathered into ~1 GiB batches: pageable pieces are first packed into
one of two reusable pinned staging buffers (already-pinned pieces are copied
directly), and each batch's H2D copy runs on a side stream while the previous
batch is being reduced.  ``threads`` is accepted for signature compatibility
(and, as in the reference, selects the fold order of "first-come").
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable

import numpy as np

from . import device as dv
from .errors import DataError, NumericalError, UsageError
from .rowchunk import RowChunk

COMBINE_ORDERS = ("tree", "sequential", "first-come")


# ---------------------------------------------------------------------------
# result types (reference tsqr.py:27-110)


@dataclass(frozen=True)
class TriangularFactor:
    """n x n upper-triangular factor with a nonnegative diagonal (read-only)."""

    entries: np.ndarray = field(repr=False)

    def __post_init__(self):
        e = self.entries
        if e.ndim != 2 or e.shape[0] != e.shape[1]:
            raise UsageError(f"triangular factor must be square, got {e.shape}")
        if np.tril(e, -1).any():
            raise UsageError("triangular factor has nonzero entries below the diagonal")
        if (np.diagonal(e) < 0).any():
            raise UsageError("triangular factor has a negative diagonal entry")
        e.setflags(write=False)

    @property
    def n(self) -> int:
        return self.entries.shape[0]

    def save(self, path):
        from .matio import write_matrix

        write_matrix(path, self.entries)
        Path(f"{path}.json").write_text(json.dumps({"kind": "triangular_factor", "n": self.n}, sort_keys=True))

    @classmethod
    def load(cls, path) -> "TriangularFactor":
        from .matio import read_matrix

        meta = json.loads(Path(f"{path}.json").read_text())
        if meta.get("kind") != "triangular_factor":
            raise DataError(f"{path} is not a saved triangular factor")
        return cls(entries=read_matrix(path))


@dataclass(frozen=True)
class ColumnStats:
    """Per-column l1 and l2 norms of the streamed matrix."""

    l1: np.ndarray = field(repr=False)
    l2: np.ndarray = field(repr=False)

    def __post_init__(self):
        self.l1.setflags(write=False)
        self.l2.setflags(write=False)

    @property
    def n(self) -> int:
        return self.l1.shape[0]

    def norms(self, kind: str) -> np.ndarray:
        if kind == "l1":
            return self.l1
        if kind == "l2":
            return self.l2
        raise UsageError(f"unknown norm kind {kind!r}")

    def save(self, path):
        from .matio import write_matrix

        write_matrix(path, np.vstack([self.l1, self.l2]))
        meta = {"kind": "column_stats", "n": self.n, "rows": ["l1", "l2"]}
        Path(f"{path}.json").write_text(json.dumps(meta, sort_keys=True))

    @classmethod
    def load(cls, path) -> "ColumnStats":
        from .matio import read_matrix

        meta = json.loads(Path(f"{path}.json").read_text())
        if meta.get("kind") != "column_stats":
            raise DataError(f"{path} is not saved column stats")
        both = read_matrix(path)
        return cls(l1=both[0].copy(), l2=both[1].copy())


@dataclass(frozen=True)
class ReducedSVD:
    singular_values: np.ndarray = field(repr=False)
    right_vectors: np.ndarray = field(repr=False)

    def reduced_matrix(self) -> np.ndarray:
        """Sigma V^T: the n x n matrix handed to column selection."""
        return self.singular_values[:, None] * self.right_vectors


@dataclass(frozen=True)
class StreamResult:
    factor: TriangularFactor
    stats: ColumnStats
    sketch: object  # projection.SketchResult | None
    rows: int
    chunks: int
    tree_depth: int


@dataclass(frozen=True)
class GramResult:
    """NEW (no reference counterpart): X^T X and column norms from one pass."""

    gram: np.ndarray = field(repr=False)
    stats: ColumnStats
    rows: int
    chunks: int
    tree_depth: int

    def __post_init__(self):
        self.gram.setflags(write=False)

    def cholesky_factor(self) -> TriangularFactor:
        """R = chol(X^T X) with the nonnegative-diagonal convention (raises
        NumericalError when the Gram matrix is not numerically positive
        definite).  Less stable than TSQR (error grows with cond(X)^2)."""
        from .errors import NumericalError

        try:
            low = np.linalg.cholesky(self.gram)
        except np.linalg.LinAlgError as exc:
            raise NumericalError(f"Gram matrix not positive definite: {exc}") from exc
        return TriangularFactor(entries=np.ascontiguousarray(low.T))


# ---------------------------------------------------------------------------
# small host-side helpers that the reference also keeps on the host


def rsvd(r: TriangularFactor, *, device: bool = False) -> ReducedSVD:
    """SVD of the n x n factor (reference tsqr.py:156-160): LAPACK on the host, or (device=True) cuSOLVER on
    the GPU (singular values to ~1e-15 relative; rows of V^T up to sign, which SPA / XRAY / NNLS ignore)."""
    if device:
        s, vt = dv.svd_reduced(r.entries)
        return ReducedSVD(singular_values=s.cpu().numpy(), right_vectors=vt.cpu().numpy())
    _, s, vt = np.linalg.svd(r.entries)
    return ReducedSVD(singular_values=s, right_vectors=vt)


def apply_column_scaling(r: TriangularFactor, stats: ColumnStats, norm_kind: str = "l1", *,
                         device: bool = False) -> TriangularFactor:
    """R D^{-1}: the factor of the column-normalised data (reference tsqr.py:163-177; device=True: the
    scaling kernel, bitwise the same quotient)."""
    norms = stats.norms(norm_kind)
    if norms.shape != (r.n,):
        raise UsageError("column stats do not match factor dimension")
    bad = np.flatnonzero(norms <= 0.0)
    if bad.size:
        raise DataError(f"column {', '.join(str(int(j)) for j in bad)} has zero norm")
    if device:
        return TriangularFactor(entries=dv.scale_columns(r.entries, norms).cpu().numpy())
    return TriangularFactor(entries=r.entries / norms)


class TreeReducer:
    """Binary-counter pairwise reduction (reference tsqr.py:201-234): pushing
    items in index order reproduces a balanced tree; ``fn(older, newer)``."""

    def __init__(self, combine_fn):
        self._fn = combine_fn
        self._levels: list = []

    def push(self, item):
        lvl = 0
        while lvl < len(self._levels) and self._levels[lvl] is not None:
            item = self._fn(self._levels[lvl], item)
            self._levels[lvl] = None
            lvl += 1
        if lvl == len(self._levels):
            self._levels.append(item)
        else:
            self._levels[lvl] = item

    def result(self):
        acc = None
        for item in self._levels:
            if item is not None:
                acc = item if acc is None else self._fn(item, acc)
        return acc

    @property
    def depth(self) -> int:
        return len(self._levels)


# ---------------------------------------------------------------------------
# single-chunk entry points


def _chunk_data(chunk):
    return chunk.data if isinstance(chunk, RowChunk) else chunk


def factor_chunk(chunk) -> TriangularFactor:
    """Sign-fixed triangular factor of one row chunk (reference tsqr.py:129-141)."""
    data = _chunk_data(chunk)
    t = dv.torch()
    if not isinstance(data, t.Tensor):
        data = np.asarray(data, dtype=np.float64)
    if data.ndim != 2 or data.shape[0] < 1:
        raise UsageError(f"chunk must have at least one row, got shape {tuple(data.shape)}")
    r, _, _ = dv.tsqr(data, stats=False)
    return TriangularFactor(entries=r.cpu().numpy())


def combine(r1: TriangularFactor, r2: TriangularFactor) -> TriangularFactor:
    """Factor of the vertical stack [r1; r2] (reference tsqr.py:144-153)."""
    if r1.n != r2.n:
        raise UsageError(f"dimension mismatch: {r1.n} vs {r2.n}")
    if not r1.entries.any():
        return r2
    if not r2.entries.any():
        return r1
    t = dv.torch()
    dev = dv.require_device()
    stack = t.from_numpy(np.stack([r1.entries, r2.entries])).to(dev)
    return TriangularFactor(entries=dv.combine_factors(stack).cpu().numpy())


# ---------------------------------------------------------------------------
# the pass


@dataclass
class _Node:
    r: object  # n x n device factor or None
    l1: object
    sq: object
    sk: object  # k x n device sketch or None
    g: object  # n x n device Gram or None
    rows: int
    n: int


def _merge_nodes(a: _Node, b: _Node) -> _Node:
    """merge_nodes of reference tsqr.py:307-311 on device tensors."""
    if a.n != b.n:
        raise UsageError(f"dimension mismatch: {a.n} vs {b.n}")
    t = dv.torch()
    r = dv.combine_factors(t.stack([a.r, b.r])) if a.r is not None else None
    sk = None
    if a.sk is not None:
        if a.sk.shape != b.sk.shape:
            raise UsageError(f"shape mismatch: {tuple(a.sk.shape)} vs {tuple(b.sk.shape)}")
        sk = a.sk + b.sk
    g = a.g + b.g if a.g is not None else None
    return _Node(r, a.l1 + b.l1, a.sq + b.sq, sk, g, a.rows + b.rows, a.n)


class _PassEngine:
    """Reduces one device row block into a _Node with the requested outputs."""

    def __init__(self, want_r: bool, sketch_rows, seed: int, want_gram: bool):
        self.want_r, self.k, self.seed, self.want_gram = want_r, sketch_rows, seed, want_gram

    def reduce(self, x, row_offset: int) -> _Node:
        m, n = int(x.shape[0]), int(x.shape[1])
        r = l1 = sq = g = sk = None
        if self.want_r:
            r, l1, sq = dv.tsqr(x, stats=True)
        if self.want_gram:
            g, gl1, gsq = dv.gram(x, stats=l1 is None)
            if l1 is None:
                l1, sq = gl1, gsq
        if l1 is None:
            l1, sq = dv.column_stats(x)
        if self.k is not None:
            sk = dv.sketch(x, row_offset, self.seed, self.k)
        return _Node(r, l1, sq, sk, g, m, n)


def _host_batches(chunks, batch_rows_for):
    """Group consecutive host chunks whose rows are contiguous into batches.
    Yields lists of (row_offset, array) pieces plus the number of input chunks
    consumed.  Oversized chunks are split into batch-sized pieces."""
    cur, cur_rows, cur_end, cur_n, consumed = [], 0, None, None, 0
    for ch in chunks:
        consumed += 1
        data = np.asarray(ch.data, dtype=np.float64) if not _is_device(ch.data) else ch.data
        if data.ndim != 2 or data.shape[0] < 1:
            raise UsageError(f"chunk must have at least one row, got shape {tuple(data.shape)}")
        n = data.shape[1]
        cap = batch_rows_for(n)
        off = int(ch.row_offset)
        pos = 0
        while pos < data.shape[0]:
            if cur and (cur_end != off + pos or cur_n != n or cur_rows >= cap):
                yield cur, consumed
                consumed = 0
                cur, cur_rows = [], 0
            take = min(cap - cur_rows, data.shape[0] - pos)
            cur.append((off + pos, data[pos:pos + take]))
            cur_rows += take
            cur_end, cur_n = off + pos + take, n
            pos += take
    if cur:
        yield cur, consumed


def _is_device(data) -> bool:
    t = dv.torch()
    return isinstance(data, t.Tensor) and data.is_cuda


HOST_BATCH_BYTES = 1 << 30  # rows per PCIe batch: ~1 GiB of X


def _device_batch(items):
    """One device matrix for consecutive device chunks with contiguous row offsets: a single strided view
    when the chunks are adjacent slices of one allocation (the usual `x[o:o + c]` pattern), else a copy."""
    t = dv.torch()
    if len(items) == 1:
        return items[0][1]
    first = items[0][1]
    ld = first.stride(0) if first.shape[0] > 1 else first.shape[1]
    adjacent = True
    ptr = first.data_ptr()
    for _, x in items:
        if x.data_ptr() != ptr or x.stride(1) != 1 or (x.shape[0] > 1 and x.stride(0) != ld):
            adjacent = False
            break
        ptr += x.shape[0] * ld * x.element_size()
    rows = sum(int(x.shape[0]) for _, x in items)
    if adjacent:
        try:
            return t.as_strided(first, (rows, first.shape[1]), (ld, 1))
        except RuntimeError:  # outside the first tensor's storage: fall back to a copy
            pass
    return t.cat([x for _, x in items], dim=0)


def _iter_nodes(chunks, engine: _PassEngine):
    """Yield (node, n_input_chunks) for the stream.  Consecutive device chunks with contiguous row offsets
    are reduced as one batch (up to ~1 GiB; a small chunk alone would occupy a fraction of the GPU —
    8192-row chunks run at 9 GB/s one by one); host chunks are batched and double-buffered over a copy
    stream.  Batching changes only the (deterministic) combination order, i.e. rounding, never the
    reported chunk count or tree depth."""
    dev = dv.require_device()
    pending_host = []
    pending_dev = []  # (row_offset, device matrix)
    dev_rows = 0

    def flush_host(items):
        yield from _reduce_host(items, engine, dev)

    def flush_dev():
        yield engine.reduce(_device_batch(pending_dev), pending_dev[0][0]), len(pending_dev)

    for ch in chunks:
        if _is_device(ch.data):
            if pending_host:
                yield from flush_host(pending_host)
                pending_host = []
            x = dv.as_device_matrix(ch.data)
            if x.shape[0] < 1:
                raise UsageError(f"chunk must have at least one row, got shape {tuple(x.shape)}")
            off = int(ch.row_offset)
            if pending_dev:
                last_off, last = pending_dev[-1]
                # adjacent slices of one allocation batch without limit (a view); others are copied, <= ~1 GiB
                ld = last.stride(0) if last.shape[0] > 1 else last.shape[1]
                adjacent = (x.data_ptr() == last.data_ptr() + last.shape[0] * ld * last.element_size()
                            and (x.shape[0] == 1 or x.stride(0) == ld))
                cap = max(1, HOST_BATCH_BYTES // (8 * int(last.shape[1])))
                if (x.shape[1] != last.shape[1] or off != last_off + int(last.shape[0])
                        or (not adjacent and dev_rows + x.shape[0] > cap)):
                    yield from flush_dev()
                    pending_dev, dev_rows = [], 0
            pending_dev.append((off, x))
            dev_rows += int(x.shape[0])
        else:
            if pending_dev:
                yield from flush_dev()
                pending_dev, dev_rows = [], 0
            pending_host.append(ch)
            if len(pending_host) >= 4096:
                yield from flush_host(pending_host)
                pending_host = []
    if pending_dev:
        yield from flush_dev()
    if pending_host:
        yield from flush_host(pending_host)


_PACK_POOL = None
_PACK_MIN_BYTES = 32 << 20  # below this one thread packs (thread hand-off costs more than it saves)


def _pack_pieces(dst: np.ndarray, arrs) -> None:
    """Copy consecutive row pieces into the pinned staging buffer, split over host threads (numpy copies
    release the GIL): one thread packs at ~8 GB/s, the PCIe copy that follows runs at ~55."""
    global _PACK_POOL
    offs = np.cumsum([0] + [a.shape[0] for a in arrs])
    total = int(offs[-1]) * dst.shape[1] * 8
    workers = min(8, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else 4)
    if total < _PACK_MIN_BYTES or workers < 2 or len(arrs) < 2:
        for a, o in zip(arrs, offs[:-1]):
            dst[o:o + a.shape[0]] = a
        return
    if _PACK_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _PACK_POOL = ThreadPoolExecutor(max_workers=workers, thread_name_prefix="tsnmf-pack")
    # contiguous groups of pieces with about equal rows
    bounds = np.searchsorted(offs, np.linspace(0, offs[-1], workers + 1)[1:-1])
    groups = np.split(np.arange(len(arrs)), bounds)

    def run(idx):
        for i in idx:
            dst[offs[i]:offs[i + 1]] = arrs[i]

    for f in [_PACK_POOL.submit(run, g) for g in groups if len(g)]:
        f.result()


def _reduce_host(chunks, engine: _PassEngine, dev):
    t = dv.torch()
    copy_stream = t.cuda.Stream(dev)
    compute_stream = t.cuda.current_stream(dev)
    bufs: list = [None, None]
    stage: list = [None, None]  # pinned host staging buffers (pageable pieces are packed here first)
    done_ev: list = [None, None]
    ready_ev: list = [None, None]
    hold: list = [None, None]  # host sources of in-flight copies
    slot = 0
    batch_rows = lambda n: max(1, HOST_BATCH_BYTES // (8 * n))  # noqa: E731
    for pieces, consumed in _host_batches(chunks, batch_rows):
        rows = sum(p[1].shape[0] for p in pieces)
        n = pieces[0][1].shape[1]
        buf = bufs[slot]
        if buf is None or buf.shape[1] != n or buf.shape[0] < rows:
            buf = t.empty((max(rows, min(batch_rows(n), 2 * rows)), n), dtype=t.float64, device=dev)
            bufs[slot] = buf
        if ready_ev[slot] is not None:
            ready_ev[slot].synchronize()  # copies two batches ago done: release their sources / staging
        hold[slot] = []
        srcs = [t.from_numpy(np.ascontiguousarray(arr)) for _, arr in pieces]
        pinned = all(s.is_pinned() for s in srcs)
        if not pinned:
            # a copy from pageable memory is staged by the driver and is effectively synchronous, so pack
            # the batch into a reusable pinned buffer: the H2D below then overlaps the previous reduction
            st = stage[slot]
            if st is None or st.shape[1] != n or st.shape[0] < rows:
                st = t.empty((buf.shape[0], n), dtype=t.float64, pin_memory=True)
                stage[slot] = st
            _pack_pieces(st.numpy(), [arr for _, arr in pieces])
            srcs = [st[:rows]]
        with t.cuda.stream(copy_stream):
            if done_ev[slot] is not None:
                copy_stream.wait_event(done_ev[slot])
            pos = 0
            for src in srcs:
                hold[slot].append(src)
                buf[pos:pos + src.shape[0]].copy_(src, non_blocking=True)
                pos += src.shape[0]
            ready = t.cuda.Event()
            ready.record(copy_stream)
        ready_ev[slot] = ready
        compute_stream.wait_event(ready)
        node = engine.reduce(buf[:rows], pieces[0][0])
        ev = t.cuda.Event()
        ev.record(compute_stream)
        done_ev[slot] = ev
        yield node, consumed
        slot ^= 1


def _run_pass(chunks, engine: _PassEngine, combine_order: str, threads: int = 1):
    if combine_order not in COMBINE_ORDERS:
        raise UsageError(f"combine_order must be one of {COMBINE_ORDERS}")
    n_chunks = 0
    depth = 0
    # reference tsqr.py:315-333: "first-come" folds in completion order only with threads > 1 (one
    # completion order of a deterministic device pass is the input order); with threads == 1 it takes the
    # ordered-map branch, i.e. the tree, and reports the tree depth
    if combine_order == "tree" or (combine_order == "first-come" and threads <= 1):
        red = TreeReducer(_merge_nodes)
        for node, consumed in _iter_nodes(chunks, engine):
            n_chunks += consumed
            red.push(node)
        node = red.result()
        depth = n_chunks.bit_length()  # TreeReducer depth over the input chunks (tsqr.py:232-234)
    else:
        node = None
        for nd, consumed in _iter_nodes(chunks, engine):
            n_chunks += consumed
            node = nd if node is None else _merge_nodes(node, nd)
    if node is None:
        raise DataError("empty chunk stream")
    return node, n_chunks, depth


def _check_square_range(l1: np.ndarray, sq: np.ndarray, stage: str) -> None:
    """The device kernels form sums of squares without LAPACK's dnrm2-style rescaling, so finite columns
    whose squares overflow (|x| >~ 1e154) or all underflow (|x| <~ 1e-154) cannot be factored faithfully;
    report them instead of returning a wrong factor.  (Known divergence: the reference's LAPACK path
    handles such magnitudes.)  Non-finite data keeps the reference's behaviour (not flagged here)."""
    bad = np.isfinite(l1) & (~np.isfinite(sq) | ((l1 > 0) & (sq == 0)))
    if bad.any():
        j = int(np.flatnonzero(bad)[0])
        raise NumericalError(f"column {j}: magnitudes outside the range where fp64 squares are representable "
                             f"(l1 = {l1[j]:.3e}, sum of squares = {sq[j]:.3e}); rescale the data", stage=stage)


def stream_pass(chunks: Iterable[RowChunk], *, sketch_rows: int | None = None, seed: int = 0,
                combine_order: str = "tree", threads: int = 1) -> StreamResult:
    """One traversal of a chunk stream: the triangular factor, the column
    norms and (with ``sketch_rows``) the Gaussian projection (reference
    tsqr.py:276-343)."""
    from .projection import SketchResult

    if combine_order not in COMBINE_ORDERS:
        raise UsageError(f"combine_order must be one of {COMBINE_ORDERS}")
    if threads < 1:
        raise UsageError(f"threads must be >= 1, got {threads}")
    if sketch_rows is not None and sketch_rows < 1:
        raise UsageError(f"sketch rows must be >= 1, got {sketch_rows}")
    node, n_chunks, depth = _run_pass(chunks, _PassEngine(True, sketch_rows, seed, False), combine_order,
                                      threads)
    if node.rows < node.n:
        raise DataError(f"not tall-and-skinny: m = {node.rows} < n = {node.n}")
    l1, sq = node.l1.cpu().numpy(), node.sq.cpu().numpy()
    _check_square_range(l1, sq, "stream_pass")
    stats = ColumnStats(l1=l1, l2=np.sqrt(sq))
    sk = SketchResult(entries=node.sk.cpu().numpy(), seed=seed) if node.sk is not None else None
    return StreamResult(factor=TriangularFactor(entries=node.r.cpu().numpy()), stats=stats, sketch=sk,
                        rows=node.rows, chunks=n_chunks, tree_depth=depth)


def gram_pass(chunks: Iterable[RowChunk], *, combine_order: str = "tree") -> GramResult:
    """NEW: one pass producing X^T X and the column norms (the BASELINE
    north-star Gram variant; no reference function)."""
    node, n_chunks, depth = _run_pass(chunks, _PassEngine(False, None, 0, True), combine_order)
    l1, sq = node.l1.cpu().numpy(), node.sq.cpu().numpy()
    _check_square_range(l1, sq, "gram_pass")
    stats = ColumnStats(l1=l1, l2=np.sqrt(sq))
    return GramResult(gram=node.g.cpu().numpy(), stats=stats, rows=node.rows, chunks=n_chunks, tree_depth=depth)


__all__ = [
    "COMBINE_ORDERS", "ColumnStats", "GramResult", "ReducedSVD", "StreamResult", "TreeReducer",
    "TriangularFactor", "apply_column_scaling", "combine", "factor_chunk", "gram_pass", "rsvd", "stream_pass",
]
