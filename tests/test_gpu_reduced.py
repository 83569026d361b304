"""Reduced-space steps on the device: GP selection (reference select.py:159-178) and column
scaling (tsqr.py:163-177, sketch.py:87-100) by this library's kernels (csrc/reduced.cu), the SVD of R
(tsqr.py:156-160) by cuSOLVER.  Compared with the live reference's golden selections and the host
restatement; the C1 chain (device R -> device rsvd -> SPA -> device NNLS) must give the reference's K and H."""
import numpy as np
import pytest

import paper_1402_6964_b200 as tb

pytestmark = pytest.mark.gpu


def test_gp_select_matches_golden(golden_select):
    for i in range(4):
        sk = golden_select[f"m{i}_sk"]
        r = len(golden_select[f"m{i}_gp"]) + int(golden_select[f"m{i}_gp_short"][0])
        ks = tb.gp_select(tb.SketchResult(sk, 0), r, device=True)
        assert list(ks.indices) == list(golden_select[f"m{i}_gp"])
        assert ks.shortfall == int(golden_select[f"m{i}_gp_short"][0])


@pytest.mark.parametrize("k,n,r,ties", [(7, 12, 4, False), (120, 200, 20, False), (400, 200, 20, True),
                                        (3, 50, 10, False), (128, 64, 16, True), (1, 700, 2, False),
                                        (40, 5000, 30, True)])
def test_gp_select_matches_host(k, n, r, ties):
    g = np.random.default_rng(k * 1000 + n)
    sk = g.integers(-3, 4, (k, n)).astype(np.float64) if ties else g.standard_normal((k, n))
    host = tb.gp_select(sk, r)
    dev = tb.gp_select(sk, r, device=True)
    assert list(dev.indices) == list(host.indices) and dev.shortfall == host.shortfall


def test_scale_columns_bitwise(golden_c1):
    st = tb.ColumnStats(np.array(golden_c1["l1"]), np.array(golden_c1["l2"]))
    sk = tb.SketchResult(np.array(golden_c1["sketch"]), 0)
    assert np.array_equal(tb.scale_columns(sk, st, device=True).entries, tb.scale_columns(sk, st).entries)
    r = tb.TriangularFactor(np.array(golden_c1["r"]))
    for kind in ("l1", "l2"):
        assert np.array_equal(tb.apply_column_scaling(r, st, kind, device=True).entries,
                              tb.apply_column_scaling(r, st, kind).entries)
    bad = tb.ColumnStats(np.where(np.arange(200) == 7, 0.0, st.l1), st.l2)
    with pytest.raises(tb.DataError):
        tb.scale_columns(sk, bad, device=True)


def test_rsvd_device(golden_c1):
    r = tb.TriangularFactor(np.array(golden_c1["r"]))
    host, dev = tb.rsvd(r), tb.rsvd(r, device=True)
    s0 = host.singular_values
    assert np.abs(dev.singular_values - s0).max() <= 1e-13 * s0[0]
    np.testing.assert_allclose(dev.singular_values, golden_c1["sigma"], rtol=1e-12, atol=1e-13 * s0[0])
    # reduced matrices agree up to the sign of each row (LAPACK's choice on either side)
    mh, md = host.reduced_matrix(), dev.reduced_matrix()
    sg = np.sign(np.sum(mh * md, axis=1))
    assert np.linalg.norm(md * sg[:, None] - mh) <= 1e-10 * np.linalg.norm(mh)


def test_c1_chain_on_device(oracle, golden_c1):
    spec = oracle.config_spec("C1")
    x = oracle.config_rows(spec, 0, spec.m)
    import torch

    res = tb.stream_pass([tb.RowChunk(0, torch.from_numpy(x).cuda())], sketch_rows=int(golden_c1["meta"][3]), seed=0)
    red = tb.rsvd(res.factor, device=True)
    k = tb.spa(red, spec.r, normalize=True, stats=res.stats)
    assert list(k.indices) == list(golden_c1["k_spa"])
    h = tb.compute_h(red, k, device=True)
    assert np.abs(h.entries - golden_c1["h_spa"]).max() <= 1e-8
    kg = tb.gp_select(tb.scale_columns(res.sketch, res.stats, device=True), spec.r, device=True)
    assert list(kg.indices) == list(golden_c1["k_gp"])
    kx = tb.xray_greedy(red, spec.r, device=True)
    assert list(kx.indices) == list(golden_c1["k_xray"])
