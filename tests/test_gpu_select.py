"""Device selection / coefficients through the C ABI (csrc/nnls.cu):
batched NNLS vs the host Lawson-Hanson (reference nnls.py:47-126) and the live reference's golden
vectors, device XRAY vs the golden selections (reference select.py:118-156), device compute_h vs the
golden H (north-star tolerance 1e-8), the C1 config end to end, and the error contract."""

import numpy as np
import pytest

import paper_1402_6964_b200 as tb
from paper_1402_6964_b200 import device as dv
from paper_1402_6964_b200 import nonneg
from paper_1402_6964_b200.errors import DataError, NumericalError, UsageError

pytestmark = pytest.mark.gpu
H_TOL = 1e-8


def test_nnls_golden(golden_select):
    a, b, y = golden_select["nnls_a"], golden_select["nnls_b"], golden_select["nnls_y"]
    got = nonneg.solve_columns(a, b[:, None], device=True)[:, 0]
    np.testing.assert_allclose(got, y, rtol=0, atol=1e-12 * max(1.0, np.abs(y).max()))


@pytest.mark.parametrize("seed,n,q,cols", [(0, 40, 6, 50), (1, 200, 20, 200), (2, 64, 33, 20), (3, 90, 64, 8)])
def test_nnls_matches_host(seed, n, q, cols):
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, 1.0, (n, q))
    ytrue = np.maximum(rng.standard_normal((q, cols)), 0.0)  # many active constraints
    b = a @ ytrue + 0.05 * rng.standard_normal((n, cols))
    host = nonneg.solve_columns(a, b)
    got = nonneg.solve_columns(a, b, device=True)
    assert np.abs(got - host).max() <= 1e-9 * max(1.0, np.abs(host).max())
    assert (got >= 0).all()
    # KKT at the device solution (reference nnls.py kkt_terms)
    for j in range(0, cols, max(1, cols // 7)):
        gmin, comp = nonneg.kkt_terms(a, b[:, j], got[:, j])
        assert gmin >= -1e-7 and comp <= 1e-7


def test_nnls_zero_and_trivial_targets():
    rng = np.random.default_rng(5)
    a = rng.uniform(0.0, 1.0, (30, 5))
    b = np.zeros((30, 3))
    b[:, 1] = -a[:, 0]  # every gradient negative: y = 0
    b[:, 2] = a[:, 3] * 2.0  # exact nonnegative fit
    y = nonneg.solve_columns(a, b, device=True)
    assert np.array_equal(y[:, 0], np.zeros(5)) and np.array_equal(y[:, 1], np.zeros(5))
    np.testing.assert_allclose(y[:, 2], [0, 0, 0, 2.0, 0], atol=1e-12)


def test_nnls_errors():
    a = np.ones((10, 3))
    with pytest.raises(UsageError):
        nonneg.solve_columns(a, np.ones((9, 2)), device=True)
    bad = np.ones((10, 2))
    bad[0, 0] = np.nan
    with pytest.raises(DataError):
        nonneg.solve_columns(a, bad, device=True)
    with pytest.raises(UsageError):
        nonneg.solve_columns(np.ones((100, dv.nnls_max_cols() + 1)), np.ones((100, 1)), device=True)
    rng = np.random.default_rng(9)
    a2 = rng.uniform(0, 1, (50, 12))
    b2 = a2 @ rng.uniform(0, 1, (12, 4))
    with pytest.raises(NumericalError) as ei:  # one iteration cannot reach the 12-variable optimum
        nonneg.solve_columns_device(a2, b2, max_iter=1)
    assert "did not converge" in str(ei.value)


@pytest.mark.parametrize("mi", [0, 1, 2, 3])
def test_xray_and_h_match_reference_golden(golden_select, mi):
    m = golden_select[f"m{mi}"]
    k_ref = list(golden_select[f"m{mi}_xray"])
    k = tb.xray_greedy(m, len(k_ref), device=True)
    assert list(k.indices) == k_ref
    h = tb.compute_h(m, k, device=True)
    assert np.abs(h.entries - golden_select[f"m{mi}_h_xray"]).max() <= H_TOL
    res = tb.relative_residual(m, k, h)
    assert abs(res - float(golden_select[f"m{mi}_res_xray"][0])) <= 1e-10


def test_c1_device_selection_matches_reference(golden_c1, oracle):
    spec = oracle.config_spec("C1")
    x = oracle.config_rows(spec, 0, spec.m)
    res = tb.stream_pass([tb.RowChunk(0, dv.torch().from_numpy(x).cuda())], sketch_rows=120, seed=0)
    red = tb.rsvd(res.factor)
    kx = tb.xray_greedy(red, 20, device=True)
    assert list(kx.indices) == list(golden_c1["k_xray"])
    k = tb.spa(red, 20, normalize=True, stats=res.stats)
    h = tb.compute_h(red, k, device=True)
    assert np.abs(h.entries - golden_c1["h_spa"]).max() <= H_TOL
    host = tb.compute_h(red, k)
    assert np.abs(h.entries - host.entries).max() <= H_TOL


def test_xray_device_usage_errors():
    m = np.random.default_rng(3).uniform(0, 1, (8, 8))
    with pytest.raises(UsageError):
        tb.xray_greedy(np.random.default_rng(1).uniform(0, 1, (80, 80)), dv.nnls_max_cols() + 1, device=True)
    with pytest.raises(UsageError):
        tb.xray_greedy(m, 9, device=True)


# ---------------------------------------------------------------------------
# Every BASELINE config's generator at a reduced row count (the full sizes are bench lines, checked by
# size-independent properties in test_gpu_fullsize.py): the device pass, selection and coefficients
# against the oracle's restatement of the reference pass on the same X.


@pytest.mark.parametrize("name,sigma,k", [("C2", None, 400), ("C3", 1e-2, 0), ("C4", None, 0), ("C5", None, 128)])
def test_config_reduced_rows_selection_matches_oracle(oracle, name, sigma, k):
    m = 1 << 17
    ospec = oracle.config_spec(name, m=m, sigma=sigma)
    x = oracle.config_rows(ospec, 0, m)
    res = tb.stream_pass([tb.RowChunk(0, dv.torch().from_numpy(x).cuda())], sketch_rows=k or None, seed=0)
    ref = oracle.stream_pass(oracle.chunks_of(x, 8192), sketch_rows=k or None, seed=0)
    r_dev, r_ref = res.factor.entries, ref.r
    assert np.linalg.norm(r_dev - r_ref) <= 1e-10 * np.linalg.norm(r_ref)
    np.testing.assert_allclose(res.stats.l1, ref.l1, rtol=1e-12)
    if k:
        assert np.linalg.norm(res.sketch.entries - ref.sketch) <= 1e-12 * np.linalg.norm(ref.sketch)
    # selection and coefficients: the device (best-iterate mode at the NNLS cap, tests/parity_full.py) vs the
    # oracle's restatement of select.py / nnls.py on its own R, never skipped
    from paper_1402_6964_b200.extremes import xray_order_device
    from paper_1402_6964_b200.nonneg import solve_columns_device

    r = ospec.r
    m_dev = tb.rsvd(res.factor).reduced_matrix()
    m_ref = oracle.reduced_matrix(r_ref)
    k_dev = list(tb.spa(m_dev, r, normalize=True, stats=res.stats).indices)
    k_ref = oracle.spa(m_ref, r, ref.l1)
    assert k_dev == k_ref
    h_dev = solve_columns_device(m_dev[:, k_dev], m_dev, capped=[])
    h_ref, _ = oracle.compute_h(m_ref, k_ref, best_effort=True)
    assert np.abs(h_dev - h_ref).max() <= H_TOL
    kx_dev = xray_order_device(m_dev, r, capped=[])
    kx_ref = oracle.xray_order(m_ref, r, best_effort=True)
    assert kx_dev == kx_ref
