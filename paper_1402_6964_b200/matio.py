"""Dense matrix files in the reference's binary layout (16-byte little-endian
header: magic b"TS", version u16 = 1, rows u64, cols u32; then row-major
float64; reference pkg/src/tsnmf/matio.py:1-25), used by the save/load
sidecars of the result types, plus a row-chunk iterator over such files.
The full reader/writer stack (text format, hashing, finiteness reports) is the
SURVEY §8f "ingest" row and is not part of this round.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import DataError
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
