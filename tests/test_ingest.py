"""ChunkReader (reference pkg/src/tsnmf/matio.py:81-156): host mode on CPU, device mode (-m gpu) against
the host mode and the oracle pass.  Messages are the reference's."""
import hashlib

import numpy as np
import pytest

import paper_1402_6964_b200 as tb
from paper_1402_6964_b200.errors import DataError, UsageError
from paper_1402_6964_b200.matio import HEADER_BYTES, ChunkReader, write_matrix


def _file(tmp_path, x, name="x.bin"):
    p = tmp_path / name
    write_matrix(p, x)
    return p


def _drain(reader):
    out = []
    for ch in reader:
        d = ch.data.cpu().numpy() if hasattr(ch.data, "cpu") else np.asarray(ch.data)
        out.append((ch.row_offset, d.copy()))
    return out


def test_host_reader_chunks_counters_hash(tmp_path):
    x = np.random.default_rng(1).uniform(0, 1, (1000, 7))
    p = _file(tmp_path, x)
    h = hashlib.sha256()
    r = ChunkReader(p, chunk_rows=300, hasher=h)
    assert (r.rows, r.cols) == (1000, 7)
    got = _drain(r)
    assert [o for o, _ in got] == [0, 300, 600, 900]
    assert np.array_equal(np.vstack([d for _, d in got]), x)
    assert r.rows_read == 1000 and r.bytes_read == HEADER_BYTES + 1000 * 7 * 8
    assert h.hexdigest() == hashlib.sha256(p.read_bytes()).hexdigest()


def test_host_reader_errors(tmp_path):
    x = np.ones((10, 3))
    p = _file(tmp_path, x)
    with pytest.raises(UsageError, match="chunk_rows must be >= 1, got 0"):
        ChunkReader(p, chunk_rows=0)
    raw = p.read_bytes()
    (tmp_path / "short.bin").write_bytes(raw[:-8])
    with pytest.raises(DataError, match="payload shorter than declared"):
        ChunkReader(tmp_path / "short.bin")
    (tmp_path / "long.bin").write_bytes(raw + b"\0" * 8)
    with pytest.raises(DataError, match="payload longer than declared"):
        ChunkReader(tmp_path / "long.bin")
    (tmp_path / "magic.bin").write_bytes(b"XX" + raw[2:])
    with pytest.raises(DataError, match="malformed header: bad magic"):
        ChunkReader(tmp_path / "magic.bin")
    (tmp_path / "hdr.bin").write_bytes(raw[:5])
    with pytest.raises(DataError, match="malformed header: file shorter than header"):
        ChunkReader(tmp_path / "hdr.bin")


def test_host_reader_nonfinite_position(tmp_path):
    x = np.random.default_rng(2).uniform(0, 1, (50, 4))
    x[23, 2] = np.nan
    x[23, 3] = np.inf
    x[40, 0] = np.inf
    p = _file(tmp_path, x)
    r = ChunkReader(p, chunk_rows=10)
    seen = []
    with pytest.raises(DataError, match=r"non-finite entry at row 23, column 2"):
        for ch in r:
            seen.append(ch.row_offset)
    assert seen == [0, 10] and r.rows_read == 20 and r.bytes_read == HEADER_BYTES + 30 * 4 * 8
    assert len(_drain(ChunkReader(p, chunk_rows=10, validate=False))) == 5


@pytest.mark.gpu
@pytest.mark.parametrize("rows,n,chunk,batch_bytes", [(10_000, 25, 8192, 1 << 30), (100_003, 200, 8192, 3 << 20),
                                                      (5000, 7, 64, 10_000)])
def test_device_reader_matches_host_and_oracle(tmp_path, oracle, rows, n, chunk, batch_bytes):
    x = np.random.default_rng(rows).uniform(0, 1, (rows, n))
    p = _file(tmp_path, x)
    hh, hd = hashlib.sha256(), hashlib.sha256()
    host = ChunkReader(p, chunk_rows=chunk, hasher=hh)
    devr = ChunkReader(p, chunk_rows=chunk, hasher=hd, device="cuda", batch_bytes=batch_bytes)
    a, b = _drain(host), _drain(devr)
    assert [o for o, _ in a] == [o for o, _ in b]
    assert all(np.array_equal(u, v) for (_, u), (_, v) in zip(a, b))
    assert (devr.rows_read, devr.bytes_read) == (host.rows_read, host.bytes_read)
    assert hd.hexdigest() == hh.hexdigest()
    res = tb.stream_pass(ChunkReader(p, chunk_rows=chunk, device="cuda", batch_bytes=batch_bytes))
    want = oracle.factor_chunk(x)
    assert np.linalg.norm(res.factor.entries - want) <= 1e-10 * np.linalg.norm(want)
    assert res.rows == rows and res.chunks == -(-rows // chunk)


@pytest.mark.gpu
@pytest.mark.parametrize("bad_row,bad_col", [(0, 0), (4095, 6), (4096, 1), (12_345, 3), (29_999, 6)])
def test_device_reader_nonfinite_like_host(tmp_path, bad_row, bad_col):
    x = np.random.default_rng(bad_row).uniform(0, 1, (30_000, 7))
    x[bad_row, bad_col] = np.nan
    if bad_row + 1 < 30_000:
        x[bad_row + 1, 0] = -np.inf  # a later bad entry must not be the one reported
    p = _file(tmp_path, x)
    outs = []
    for dev in (None, "cuda"):
        r = ChunkReader(p, chunk_rows=1000, device=dev, batch_bytes=7 * 8 * 4096)
        seen = []
        with pytest.raises(DataError) as e:
            for ch in r:
                seen.append(ch.row_offset)
        outs.append((str(e.value), seen, r.rows_read, r.bytes_read))
    assert outs[0] == outs[1]
    assert f"row {bad_row}, column {bad_col}" in outs[0][0]


@pytest.mark.gpu
def test_device_reader_edge_cases(tmp_path):
    """Empty payload (the pass reports the reference's empty-stream error), validation off (NaN passes
    through to the factor as in the reference), a single short batch."""
    p0 = _file(tmp_path, np.zeros((0, 5)), "empty.bin")
    assert _drain(ChunkReader(p0, device="cuda")) == []
    with pytest.raises(DataError, match="empty chunk stream"):
        tb.stream_pass(ChunkReader(p0, device="cuda"))
    x = np.random.default_rng(3).uniform(0, 1, (777, 9))
    x[5, 5] = np.nan
    p1 = _file(tmp_path, x, "nan.bin")
    got = _drain(ChunkReader(p1, chunk_rows=100, device="cuda", validate=False))
    assert np.isnan(np.vstack([d for _, d in got])[5, 5]) and len(got) == 8


def test_gds_needs_a_device(tmp_path):
    p = _file(tmp_path, np.ones((4, 3)))
    with pytest.raises(UsageError, match="gds=True needs device="):
        ChunkReader(p, gds=True)


def test_cufile_binding_loads_or_reports():
    """The cuFile binding is optional: either libcufile loads and exports the calls used, or available() is
    False (and ChunkReader(gds=True) raises at iteration time, tested on the GPU)."""
    from paper_1402_6964_b200 import gds

    if gds.available():
        lib = gds._load()
        for name in ("cuFileDriverOpen", "cuFileHandleRegister", "cuFileHandleDeregister", "cuFileRead"):
            assert hasattr(lib, name)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,n,chunk,batch_bytes", [(10_000, 25, 8192, 1 << 30), (100_003, 200, 8192, 3 << 20),
                                                      (5000, 7, 64, 10_000)])
def test_gds_reader_matches_host_and_oracle(tmp_path, oracle, rows, n, chunk, batch_bytes):
    """cuFile path (GPUDirect Storage where the box has it, libcufile's compatibility mode elsewhere): same
    chunks, offsets and counters as the host reader, and the pass over it matches the oracle."""
    from paper_1402_6964_b200 import gds

    if not gds.usable():
        pytest.skip(f"cuFile is not usable on this box: {gds.usable_reason()}")
    x = np.random.default_rng(rows + 1).uniform(0, 1, (rows, n))
    p = _file(tmp_path, x)
    host = ChunkReader(p, chunk_rows=chunk)
    devr = ChunkReader(p, chunk_rows=chunk, device="cuda", batch_bytes=batch_bytes, gds=True)
    a, b = _drain(host), _drain(devr)
    assert [o for o, _ in a] == [o for o, _ in b]
    assert all(np.array_equal(u, v) for (_, u), (_, v) in zip(a, b))
    assert (devr.rows_read, devr.bytes_read) == (host.rows_read, host.bytes_read)
    res = tb.stream_pass(ChunkReader(p, chunk_rows=chunk, device="cuda", batch_bytes=batch_bytes, gds=True),
                         sketch_rows=8, seed=3)
    want = oracle.stream_pass(oracle.chunks_of(x, chunk), sketch_rows=8, seed=3)
    assert np.linalg.norm(res.factor.entries - want.r) <= 1e-10 * np.linalg.norm(want.r)
    assert np.linalg.norm(res.sketch.entries - want.sketch) <= 1e-12 * np.linalg.norm(want.sketch)
    assert res.rows == rows and res.chunks == -(-rows // chunk)
    # a hashed run keeps the pinned-buffer path (the hash is defined over host bytes) and still hashes the file
    h = hashlib.sha256()
    _drain(ChunkReader(p, chunk_rows=chunk, device="cuda", batch_bytes=batch_bytes, gds=True, hasher=h))
    assert h.hexdigest() == hashlib.sha256(p.read_bytes()).hexdigest()


@pytest.mark.gpu
@pytest.mark.parametrize("bad_row,bad_col", [(0, 0), (4096, 1), (29_999, 6)])
def test_gds_reader_nonfinite_like_host(tmp_path, bad_row, bad_col):
    from paper_1402_6964_b200 import gds

    if not gds.usable():
        pytest.skip(f"cuFile is not usable on this box: {gds.usable_reason()}")
    x = np.random.default_rng(bad_row).uniform(0, 1, (30_000, 7))
    x[bad_row, bad_col] = np.inf
    p = _file(tmp_path, x)
    outs = []
    for kw in ({}, {"device": "cuda", "gds": True}):
        r = ChunkReader(p, chunk_rows=1000, batch_bytes=7 * 8 * 4096, **kw)
        seen = []
        with pytest.raises(DataError) as e:
            for ch in r:
                seen.append(ch.row_offset)
        outs.append((str(e.value), seen, r.rows_read, r.bytes_read))
    assert outs[0] == outs[1]
    assert f"row {bad_row}, column {bad_col}" in outs[0][0]


@pytest.mark.gpu
def test_gds_reader_reports_an_unusable_driver(tmp_path):
    """Where libcufile is missing or its driver does not open (this pool's boxes: cuFileDriverOpen never
    returns without nvidia-fs), gds=True fails loudly instead of hanging or falling back silently."""
    from paper_1402_6964_b200 import gds
    from paper_1402_6964_b200.errors import TsnmfError

    if gds.usable():
        pytest.skip("cuFile works here; the usable path is tested above")
    p = _file(tmp_path, np.ones((64, 3)))
    with pytest.raises(TsnmfError, match="cuFile"):
        _drain(ChunkReader(p, device="cuda", gds=True))
