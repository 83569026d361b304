"""Host-side logic of the product: selection / NNLS against the reference's
golden outputs, result-type validation, tree order, chunk batching, sharding
arithmetic, matrix files.  CPU only."""

import numpy as np
import pytest

import paper_1402_6964_b200 as tb
from paper_1402_6964_b200 import extremes, factor, nonneg, sharded


@pytest.mark.parametrize("i", range(4))
def test_selection_matches_reference(golden_select, i):
    g = golden_select
    rr = g[f"m{i}"]
    r = 4 if i < 2 else 8
    stats = tb.ColumnStats(l1=g[f"m{i}_l1"].copy(), l2=np.ones_like(g[f"m{i}_l1"]))
    assert list(tb.spa(rr, r, normalize=True, stats=stats).indices) == list(g[f"m{i}_spa"])
    assert list(tb.spa(rr, r).indices) == list(g[f"m{i}_spa_raw"])
    kx = tb.xray_greedy(rr, r)
    assert list(kx.indices) == list(g[f"m{i}_xray"])
    h = tb.compute_h(rr, kx)
    np.testing.assert_allclose(h.entries, g[f"m{i}_h_xray"], atol=1e-10)
    assert abs(tb.relative_residual(rr, kx, h) - g[f"m{i}_res_xray"][0]) < 1e-12
    gp = tb.gp_select(tb.SketchResult(entries=g[f"m{i}_sk"].copy(), seed=0), r)
    assert list(gp.indices) == list(g[f"m{i}_gp"]) and gp.shortfall == g[f"m{i}_gp_short"][0]


def test_nnls_matches_reference(golden_select):
    y = tb.nnls_solve(golden_select["nnls_a"], golden_select["nnls_b"])
    np.testing.assert_allclose(y, golden_select["nnls_y"], atol=1e-12)
    gmin, comp = tb.kkt_terms(golden_select["nnls_a"], golden_select["nnls_b"], y)
    assert gmin >= -1e-8 and comp <= 1e-8 * np.dot(golden_select["nnls_b"], golden_select["nnls_b"])


def test_c1_selection_on_reference_factor(golden_c1):
    """The host selection + NNLS reproduce the reference on the reference's own R."""
    r = tb.TriangularFactor(entries=golden_c1["r"].copy())
    stats = tb.ColumnStats(l1=golden_c1["l1"].copy(), l2=golden_c1["l2"].copy())
    red = tb.rsvd(r)
    k = tb.spa(red, 20, normalize=True, stats=stats)
    assert list(k.indices) == list(golden_c1["k_spa"])
    h = tb.compute_h(red, k)
    assert np.abs(h.entries - golden_c1["h_spa"]).max() <= 1e-8
    assert list(tb.xray_greedy(red, 20).indices) == list(golden_c1["k_xray"])
    sk = tb.scale_columns(tb.SketchResult(entries=golden_c1["sketch"].copy(), seed=0), stats)
    assert list(tb.gp_select(sk, 20).indices) == list(golden_c1["k_gp"])


def test_spec_selection_toys():
    # SPEC examples: identity -> picks in order; rank errors
    assert tb.spa(np.eye(3), 3).indices == (0, 1, 2)
    with pytest.raises(tb.UsageError):
        tb.spa(np.eye(3), 4)
    with pytest.raises(tb.UsageError):
        tb.xray_greedy(np.eye(3), 0)
    with pytest.raises(tb.NumericalError) as e:
        tb.spa(np.array([[1.0, 2.0], [0.0, 0.0]]), 2)
    assert e.value.achieved == 1
    gp = tb.gp_select(np.array([[0.0, 1.0, 2.0]]), 3)
    assert gp.indices == (0, 2) and gp.shortfall == 1
    with pytest.raises(tb.UsageError):
        tb.compute_h(np.eye(3), [])


def test_result_type_validation():
    with pytest.raises(tb.UsageError):
        tb.TriangularFactor(entries=np.array([[1.0, 0], [1.0, 1.0]]))
    with pytest.raises(tb.UsageError):
        tb.TriangularFactor(entries=np.diag([1.0, -1.0]))
    f = tb.TriangularFactor(entries=np.diag([1.0, -0.0]))
    assert not f.entries.flags.writeable
    with pytest.raises(tb.DataError):
        tb.SketchResult(entries=np.array([[np.nan]]), seed=0)
    with pytest.raises(tb.UsageError):
        tb.merge_sketches(tb.SketchResult(np.ones((2, 2)), 1), tb.SketchResult(np.ones((2, 2)), 2))
    s = tb.scale_columns(tb.SketchResult(np.array([[2.0, 4.0]]), 0), tb.ColumnStats(np.array([2.0, 4.0]),
                                                                                     np.ones(2)))
    assert np.array_equal(s.entries, [[1.0, 1.0]])
    r = tb.apply_column_scaling(tb.TriangularFactor(np.diag([5.0, 10.0])),
                                tb.ColumnStats(np.array([5.0, 10.0]), np.ones(2)))
    assert np.array_equal(r.entries, np.eye(2))
    with pytest.raises(tb.DataError):
        tb.apply_column_scaling(tb.TriangularFactor(np.eye(2)), tb.ColumnStats(np.array([1.0, 0.0]), np.ones(2)))
    assert tb.default_sketch_rows(20) == 120


def test_combine_zero_operand_is_identity_without_device():
    a = tb.TriangularFactor(entries=np.diag([3.0, 4.0]))
    z = tb.TriangularFactor(entries=np.zeros((2, 2)))
    assert tb.combine(a, z) is a and tb.combine(z, a) is a
    with pytest.raises(tb.UsageError):
        tb.combine(a, tb.TriangularFactor(entries=np.eye(3)))


def test_tree_reducer_order_matches_reference(oracle):
    """fn(older, newer) over a binary-counter tree, identical to tsqr.py:201-234."""
    for count in range(1, 40):
        mine = factor.TreeReducer(lambda a, b: f"({a}+{b})")
        ref = oracle.TreeReducer(lambda a, b: f"({a}+{b})")
        for i in range(count):
            mine.push(str(i))
            ref.push(str(i))
        assert mine.result() == ref.result() and mine.depth == ref.depth == count.bit_length()


def test_host_batching_groups_contiguous_chunks():
    x = np.arange(40.0).reshape(20, 2)
    chunks = [tb.RowChunk(o, x[o:o + 3]) for o in range(0, 20, 3)]
    batches = list(factor._host_batches(chunks, lambda n: 8))
    pieces = [p for b, _ in batches for p in b]
    assert sum(c for _, c in batches) == len(chunks)
    assert np.array_equal(np.vstack([a for _, a in pieces]), x)
    for b, _ in batches:
        rows = sum(a.shape[0] for _, a in b)
        assert rows <= 8
        offs = [o for o, _ in b]
        ends = [o + a.shape[0] for o, a in b]
        assert offs[1:] == ends[:-1]
    # non-contiguous offsets start a new batch
    gap = [tb.RowChunk(0, x[:2]), tb.RowChunk(10, x[2:4])]
    assert len(list(factor._host_batches(gap, lambda n: 100))) == 2
    with pytest.raises(tb.UsageError):
        list(factor._host_batches([tb.RowChunk(0, np.ones(3))], lambda n: 8))


def test_shard_ranges_cover_rows():
    for m in (1, 7, 100, 2**26 + 3):
        for world in (1, 2, 3, 4, 8):
            spans = [sharded.shard_range(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_matrix_file_roundtrip(tmp_path):
    a = np.random.default_rng(0).standard_normal((7, 3))
    tb.write_matrix(tmp_path / "a.tsm", a)
    assert np.array_equal(tb.read_matrix(tmp_path / "a.tsm"), a)
    f = tb.TriangularFactor(entries=np.triu(np.abs(a[:3])))
    f.save(tmp_path / "R.tsm")
    assert np.array_equal(tb.TriangularFactor.load(tmp_path / "R.tsm").entries, f.entries)
    (tmp_path / "bad.tsm").write_bytes(b"XX" + bytes(30))
    with pytest.raises(tb.DataError):
        tb.read_matrix(tmp_path / "bad.tsm")
    from paper_1402_6964_b200 import matio

    chunks = list(matio.iter_chunks(tmp_path / "a.tsm", 3))
    assert [c.row_offset for c in chunks] == [0, 3, 6]


def test_sweep_host(golden_select):
    rr = golden_select["m2"]
    stats = tb.ColumnStats(l1=golden_select["m2_l1"].copy(), l2=np.ones(rr.shape[1]))
    rep = tb.sweep(rr, stats, ["spa", "xray"], range(1, 9))
    res = rep.residuals("spa")
    assert all(res[r + 1] <= res[r] + 1e-12 for r in range(1, 8))
    assert rep.to_json_dict()["cells"][0]["algorithm"] == "spa"
    with pytest.raises(tb.UsageError):
        tb.sweep(rr, stats, ["gp"], [1])


def test_sweep_report_files(golden_select, tmp_path):
    import csv
    import json

    rr = golden_select["m2"]
    stats = tb.ColumnStats(l1=golden_select["m2_l1"].copy(), l2=np.ones(rr.shape[1]))
    rep = tb.sweep(rr, stats, ["spa"], range(1, 4))
    rep.write_json(tmp_path / "s.json")
    rep.write_csv(tmp_path / "s.csv")
    assert json.loads((tmp_path / "s.json").read_text()) == rep.to_json_dict()
    rows = list(csv.reader(open(tmp_path / "s.csv")))
    assert rows[0] == ["r", "algorithm", "residual", "seconds"] and len(rows) == 4
    assert [float(r[2]) for r in rows[1:]] == [rep.residuals("spa")[r] for r in (1, 2, 3)]


def test_gram_result_cholesky():
    from paper_1402_6964_b200.factor import GramResult

    x = np.random.default_rng(3).standard_normal((500, 12))
    g = GramResult(gram=x.T @ x, stats=tb.ColumnStats(l1=np.abs(x).sum(0), l2=np.sqrt((x * x).sum(0))),
                   rows=500, chunks=1, tree_depth=1)
    r = g.cholesky_factor().entries
    q = np.linalg.qr(x, mode="r")
    q = q * np.sign(np.diagonal(q))[:, None]
    assert np.abs(r - q).max() <= 1e-10 * np.abs(q).max()
    bad = GramResult(gram=-np.eye(3), stats=tb.ColumnStats(l1=np.ones(3), l2=np.ones(3)), rows=3, chunks=1,
                     tree_depth=1)
    with pytest.raises(tb.NumericalError):
        bad.cholesky_factor()


def test_nnls_input_checks():
    with pytest.raises(tb.UsageError):
        nonneg.nnls_solve(np.ones((3, 2)), np.ones(4))
    with pytest.raises(tb.DataError):
        nonneg.nnls_solve(np.array([[np.inf]]), np.ones(1))
    y = nonneg.nnls_solve(np.eye(2), np.array([1.0, -1.0]))
    assert np.array_equal(y, [1.0, 0.0])
    assert extremes.as_matrix(tb.TriangularFactor(np.eye(2))).shape == (2, 2)


def test_square_range_check():
    """Columns whose squares overflow or all underflow are reported (the device kernels do not rescale);
    zero and non-finite columns are left to the reference's own handling."""
    import numpy as np
    import pytest

    from paper_1402_6964_b200.errors import NumericalError
    from paper_1402_6964_b200.factor import _check_square_range

    _check_square_range(np.array([1.0, 0.0, np.nan]), np.array([1.0, 0.0, np.nan]), "t")
    with pytest.raises(NumericalError, match="column 1"):
        _check_square_range(np.array([1.0, 1e-160]), np.array([1.0, 0.0]), "t")
    with pytest.raises(NumericalError, match="column 0"):
        _check_square_range(np.array([1e200]), np.array([np.inf]), "t")


def test_default_sketch_rows():
    """k = ceil(2 r ln max(r, 2)) (reference sketch.py:57-59; values from the live reference)."""
    from paper_1402_6964_b200.projection import default_sketch_rows

    assert [default_sketch_rows(r) for r in (1, 2, 3, 10, 20, 64)] == [2, 3, 7, 47, 120, 533]


def test_pack_pieces_parallel_matches_vstack(monkeypatch):
    """Host chunks are packed into the pinned staging buffer by several threads (factor._pack_pieces)."""
    from paper_1402_6964_b200 import factor as f

    monkeypatch.setattr(f, "_PACK_MIN_BYTES", 0)
    g = np.random.default_rng(1)
    for sizes in ([1], [3, 7, 8192, 100, 1, 4000], [5] * 37, [100_000, 3]):
        arrs = [g.standard_normal((r, 9)) for r in sizes]
        dst = np.zeros((sum(sizes) + 5, 9))
        f._pack_pieces(dst, arrs)
        assert np.array_equal(dst[:sum(sizes)], np.vstack(arrs)) and not dst[sum(sizes):].any()
