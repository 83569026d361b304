"""Dense matrix files in the reference's binary layout (16-byte little-endian
header: magic b"TS", version u16 = 1, rows u64, cols u32; then row-major
float64; reference pkg/src/tsnmf/matio.py:1-25): read_matrix / write_matrix for
the result types' sidecars, and ChunkReader — the reference's streaming reader
(matio.py:90-156: same parameters, counters, content hashing and errors) with a
device mode that feeds the B200 pass: large sequential reads
into pinned buffers, copies on a side stream, the finiteness check on the device.
The text format is not mirrored.
"""

from __future__ import annotations

import os
import struct
from pathlib import Path

import numpy as np

from .errors import DataError, UsageError
from .rowchunk import RowChunk

_HDR = struct.Struct("<2sHQI")
HEADER_BYTES = _HDR.size


def write_matrix(path, a) -> None:
    a = np.ascontiguousarray(np.asarray(a, dtype="<f8"))
    if a.ndim != 2:
        raise DataError(f"expected a 2-D matrix, got shape {a.shape}")
    with open(path, "wb") as f:
        f.write(_HDR.pack(b"TS", 1, a.shape[0], a.shape[1]))
        f.write(a.tobytes())


def _header(raw: bytes, path) -> tuple[int, int]:
    if len(raw) < HEADER_BYTES:
        raise DataError(f"{path}: malformed header: file shorter than header")
    magic, version, rows, cols = _HDR.unpack(raw[:HEADER_BYTES])
    if magic != b"TS":
        raise DataError(f"{path}: malformed header: bad magic")
    if version != 1:
        raise DataError(f"{path}: malformed header: unsupported version {version}")
    if cols < 1:
        raise DataError(f"{path}: matrix must have at least one column")
    return rows, cols


def read_matrix(path) -> np.ndarray:
    raw = Path(path).read_bytes()
    rows, cols = _header(raw, path)
    body = raw[HEADER_BYTES:]
    if len(body) != rows * cols * 8:
        raise DataError(f"{path}: payload is {len(body)} bytes, expected {rows * cols * 8}")
    return np.frombuffer(body, dtype="<f8").reshape(rows, cols).astype(np.float64)


def iter_chunks(path, chunk_rows: int = 8192):
    """RowChunks of a matrix file (memory-mapped; host chunks)."""
    with open(path, "rb") as f:
        rows, cols = _header(f.read(HEADER_BYTES), path)
    mm = np.memmap(path, dtype="<f8", mode="r", offset=HEADER_BYTES, shape=(rows, cols))
    for off in range(0, rows, chunk_rows):
        yield RowChunk(row_offset=off, data=np.asarray(mm[off:off + chunk_rows]))


DEFAULT_CHUNK_ROWS = 8192  # reference matio.py:27


def _unpack_header_ref(raw: bytes) -> tuple[int, int]:
    """Header checks with the reference's messages (matio.py:54-62, MatrixHeader :40-46)."""
    if len(raw) < HEADER_BYTES:
        raise DataError("malformed header: file shorter than header")
    magic, version, rows, cols = _HDR.unpack(raw[:HEADER_BYTES])
    if magic != b"TS":
        raise DataError("malformed header: bad magic")
    if version != 1:
        raise DataError(f"malformed header: unsupported version {version}")
    if cols < 1:
        raise DataError(f"matrix must have at least one column, got {cols}")
    return rows, cols


def _nonfinite_error(block_row0: int, row_in_block: int, col: int) -> DataError:
    # reference matio.py:81-87
    return DataError(f"non-finite entry at row {block_row0 + row_in_block}, column {col}")


class ChunkReader:
    """Streams RowChunks from a binary matrix file (reference matio.py:90-156).

    Parameters and attributes follow the reference: ``chunk_rows`` (rows per chunk, the last may be
    shorter), ``validate`` (reject NaN/Inf, reporting the first bad row and column), ``hasher``
    (hashlib-style object updated with every byte read, header included), ``rows_read`` /
    ``bytes_read`` counters, and the same DataError / UsageError messages.

    ``device`` (new): a CUDA device (``"cuda"``, ``torch.device`` or index) makes the reader yield
    device-resident chunks.  Whole chunks are read in batches of ~``batch_bytes`` into one of two
    pinned host buffers, copied to the device on a side stream (overlapping the consumer's kernels on
    the current stream), validated on the device (``tsnmf_first_nonfinite``: one HBM sweep per batch),
    and yielded as row views of the batch, so ``stream_pass`` reduces consecutive chunks as one batch.
    Chunk boundaries, order, counters, hash and error positions are those of the host reader: chunks
    before a non-finite entry are yielded, the error is raised when its chunk is reached.

    ``gds`` (new, device mode only): read the batches with cuFile (GPUDirect Storage, ``gds.py``) straight
    into device batches, a read-ahead thread issuing the next ``cuFileRead`` while the current batch is
    consumed; no host copy of the payload exists, so it applies when no ``hasher`` is given
    (the content hash is defined over host bytes; a hashed run keeps the pinned-buffer path).  ``None``
    follows the environment (``TSNMF_GDS=1``); ``True`` raises ``TsnmfError`` when libcufile is missing.
    """

    def __init__(self, path, chunk_rows: int = DEFAULT_CHUNK_ROWS, *, validate: bool = True, hasher=None,
                 device=None, batch_bytes: int = 1 << 30, gds: bool | None = None):
        if chunk_rows < 1:
            raise UsageError(f"chunk_rows must be >= 1, got {chunk_rows}")
        self.path = Path(path)
        self.chunk_rows = chunk_rows
        self.validate = validate
        self.hasher = hasher
        self.device = device
        self.batch_bytes = int(batch_bytes)
        if gds and device is None:
            raise UsageError("gds=True needs device= (cuFile reads into device memory)")
        self.gds = gds
        self.rows_read = 0
        self.bytes_read = 0
        size = self.path.stat().st_size
        with open(self.path, "rb") as f:
            raw = f.read(HEADER_BYTES)
        self._rows, self._cols = _unpack_header_ref(raw)
        expected = HEADER_BYTES + self._rows * self._cols * 8
        if size < expected:
            raise DataError("payload shorter than declared")
        if size > expected:
            raise DataError("payload longer than declared")

    @property
    def rows(self) -> int:
        return self._rows

    @property
    def cols(self) -> int:
        return self._cols

    def __iter__(self):
        if self.device is None:
            return self._iter_host()
        gds = self.gds if self.gds is not None else os.environ.get("TSNMF_GDS", "0") not in ("", "0")
        if gds and self.hasher is None:
            return self._iter_device_gds()
        return self._iter_device()

    def _read_header(self, f) -> None:
        raw = f.read(HEADER_BYTES)
        if self.hasher is not None:
            self.hasher.update(raw)
        self.bytes_read += len(raw)

    def _iter_host(self):
        n = self._cols
        with open(self.path, "rb") as f:
            self._read_header(f)
            offset = 0
            while offset < self._rows:
                c = min(self.chunk_rows, self._rows - offset)
                raw = f.read(c * n * 8)
                if len(raw) < c * n * 8:
                    raise DataError("payload shorter than declared")
                if self.hasher is not None:
                    self.hasher.update(raw)
                self.bytes_read += len(raw)
                block = np.frombuffer(raw, dtype="<f8").reshape(c, n)
                if self.validate and not np.isfinite(block).all():
                    bad = np.argwhere(~np.isfinite(block))[0]
                    raise _nonfinite_error(offset, int(bad[0]), int(bad[1]))
                self.rows_read += c
                yield RowChunk(row_offset=offset, data=block)
                offset += c

    def _iter_device(self):
        from . import device as dv

        t = dv.torch()
        dev = t.device(self.device) if not isinstance(self.device, int) else t.device("cuda", self.device)
        if dev.type != "cuda":
            raise UsageError(f"ChunkReader device must be a CUDA device, got {self.device!r}")
        if dev.index is None:
            dev = t.device("cuda", t.cuda.current_device())
        n = self._cols
        row_bytes = n * 8
        per_batch = max(1, self.batch_bytes // (row_bytes * self.chunk_rows)) * self.chunk_rows
        per_batch = min(per_batch, max(self._rows, 1))
        host = [t.empty((per_batch, n), dtype=t.float64).pin_memory() for _ in range(2)]
        views = [memoryview(h.numpy()).cast("B") for h in host]
        copy_stream = t.cuda.Stream(dev)
        compute = t.cuda.current_stream(dev)
        batches = [(o, min(per_batch, self._rows - o)) for o in range(0, self._rows, per_batch)]
        from concurrent.futures import ThreadPoolExecutor

        with open(self.path, "rb") as f, ThreadPoolExecutor(max_workers=1) as pool:
            self._read_header(f)

            def read_into(k, rows):  # worker thread: sequential reads (the GIL is released while reading)
                return f.readinto(views[k][:rows * row_bytes])

            # read-ahead: batch i+1 is read into the other pinned buffer while batch i is copied, scanned and
            # consumed; that buffer's previous copy finished at the scan's synchronisation point
            pending = pool.submit(read_into, 0, batches[0][1]) if batches else None
            for i, (offset, rows) in enumerate(batches):
                k = i & 1
                got = pending.result()
                view = views[k]
                if got < rows * row_bytes:
                    # the reference reads chunk by chunk: account for the whole chunks it would deliver
                    self._account(view, got // (self.chunk_rows * row_bytes) * self.chunk_rows, offset, n)
                    raise DataError("payload shorter than declared")
                hb = host[k][:rows]
                with t.cuda.stream(copy_stream):  # copy + device scan: only this stream is waited on
                    xb = t.empty((rows, n), dtype=t.float64, device=dev)
                    xb.copy_(hb, non_blocking=True)
                    ev = t.cuda.Event()
                    ev.record(copy_stream)
                    bad = dv.first_nonfinite(xb) if self.validate else -1
                    if not self.validate:
                        ev.synchronize()  # host buffer k is refilled next: its copy must be done
                compute.wait_event(ev)
                xb.record_stream(compute)
                if i + 1 < len(batches):
                    pending = pool.submit(read_into, k ^ 1, batches[i + 1][1])
                good_rows = rows if bad < 0 else (bad // n)
                for r0 in range(0, rows, self.chunk_rows):
                    c = min(self.chunk_rows, rows - r0)
                    raw = view[r0 * row_bytes:(r0 + c) * row_bytes]
                    if self.hasher is not None:
                        self.hasher.update(raw)
                    self.bytes_read += len(raw)
                    if bad >= 0 and r0 + c > good_rows:
                        raise _nonfinite_error(offset + r0, good_rows - r0, int(bad % n))
                    self.rows_read += c
                    yield RowChunk(row_offset=offset + r0, data=xb[r0:r0 + c])

    def _iter_device_gds(self):
        """cuFile path: file -> device batches without a host copy (see the class docstring)."""
        from concurrent.futures import ThreadPoolExecutor

        from . import device as dv
        from . import gds

        t = dv.torch()
        dev = t.device(self.device) if not isinstance(self.device, int) else t.device("cuda", self.device)
        if dev.type != "cuda":
            raise UsageError(f"ChunkReader device must be a CUDA device, got {self.device!r}")
        if dev.index is None:
            dev = t.device("cuda", t.cuda.current_device())
        n = self._cols
        row_bytes = n * 8
        per_batch = max(1, self.batch_bytes // (row_bytes * self.chunk_rows)) * self.chunk_rows
        per_batch = min(per_batch, max(self._rows, 1))
        batches = [(o, min(per_batch, self._rows - o)) for o in range(0, self._rows, per_batch)]
        compute = t.cuda.current_stream(dev)
        self.bytes_read += HEADER_BYTES  # the header was read (and checked) by the constructor
        with gds.FileHandle(self.path) as fh, ThreadPoolExecutor(max_workers=1) as pool:

            def read_into(xb, ready, offset, rows):  # worker thread: blocking cuFileRead into a device batch
                # cuFileRead is not stream-ordered: the batch's memory may be a block the caching allocator
                # took back from an earlier batch whose kernels are still running on the consumer's stream
                ready.synchronize()
                with t.cuda.device(dev):
                    return fh.read_into(xb.data_ptr(), rows * row_bytes, HEADER_BYTES + offset * row_bytes)

            def submit(offset, rows):
                # a fresh device batch per read (the consumer keeps views of earlier batches until it has
                # launched their reduction); the read of batch i + 2 so overlaps the reduction of batch i
                with t.cuda.device(dev):
                    xb = t.empty((rows, n), dtype=t.float64, device=dev)
                    ready = t.cuda.Event()
                    ready.record(compute)
                return xb, pool.submit(read_into, xb, ready, offset, rows)

            nxt = submit(*batches[0]) if batches else None
            for i, (offset, rows) in enumerate(batches):
                xb, fut = nxt
                got = fut.result()
                nxt = submit(*batches[i + 1]) if i + 1 < len(batches) else None
                if got < rows * row_bytes:
                    whole = got // (self.chunk_rows * row_bytes) * self.chunk_rows
                    self.rows_read += whole
                    self.bytes_read += whole * row_bytes
                    raise DataError("payload shorter than declared")
                bad = dv.first_nonfinite(xb) if self.validate else -1
                good_rows = rows if bad < 0 else (bad // n)
                for r0 in range(0, rows, self.chunk_rows):
                    c = min(self.chunk_rows, rows - r0)
                    self.bytes_read += c * row_bytes
                    if bad >= 0 and r0 + c > good_rows:
                        raise _nonfinite_error(offset + r0, good_rows - r0, int(bad % n))
                    self.rows_read += c
                    yield RowChunk(row_offset=offset + r0, data=xb[r0:r0 + c])

    def _account(self, view, whole_rows: int, offset: int, n: int) -> None:
        """Counters and hash for the whole chunks read before a short payload (reference behaviour)."""
        row_bytes = n * 8
        for r0 in range(0, whole_rows, self.chunk_rows):
            raw = view[r0 * row_bytes:(r0 + self.chunk_rows) * row_bytes]
            if self.hasher is not None:
                self.hasher.update(raw)
            self.bytes_read += len(raw)
            self.rows_read += self.chunk_rows
