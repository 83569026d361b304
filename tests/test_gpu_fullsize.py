"""Size-independent properties at BASELINE-scale row counts (m = 2^24 x 200 fp64 = 27 GB resident;
the oracle cannot run here, so parity is through invariants):
  * Gram equivalence  ||R^T R - X^T X|| <= 1e-10 ||X^T X||   (reference SPEC.md:164)
  * chunk / split invariance: R(X) == combine(R(top), R(bottom)) to 1e-12
  * stats: TSQR-fused l1 / sumsq == standalone kernel == Gram diagonal
  * sketch linearity over row splits with the global row offset (reference sketch.py:62-84)
  * R shape invariants (upper triangular, nonnegative diagonal)."""

import numpy as np
import pytest
import torch

import paper_1402_6964_b200 as tb
from conftest import rel_err
from paper_1402_6964_b200 import device as dv
from paper_1402_6964_b200 import synthetic

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
M = 1 << 24


@pytest.fixture(scope="module")
def x_big():
    spec = synthetic.config("C2", m=M)
    x = synthetic.generate(spec)
    yield x
    del x
    torch.cuda.empty_cache()


def test_fullsize_invariants(x_big):
    m, n = x_big.shape
    r, l1, sq = dv.tsqr(x_big)
    g, gl1, gsq = dv.gram(x_big)
    r, g = r.cpu().numpy(), g.cpu().numpy()
    assert np.array_equal(np.tril(r, -1), np.zeros_like(r)) and (np.diagonal(r) >= 0).all()
    assert rel_err(r.T @ r, g) <= 1e-10
    sl1, ssq = dv.column_stats(x_big)
    np.testing.assert_allclose(l1.cpu().numpy(), sl1.cpu().numpy(), rtol=1e-12)
    np.testing.assert_allclose(gl1.cpu().numpy(), sl1.cpu().numpy(), rtol=1e-12)
    np.testing.assert_allclose(sq.cpu().numpy(), np.diagonal(g), rtol=1e-12)
    np.testing.assert_allclose(ssq.cpu().numpy(), np.diagonal(g), rtol=1e-12)


def test_fullsize_split_invariance(x_big):
    m = x_big.shape[0]
    h = m // 2 + 12345  # uneven split
    whole = tb.stream_pass([tb.RowChunk(0, x_big)], sketch_rows=64, seed=3)
    parts = tb.stream_pass([tb.RowChunk(0, x_big[:h]), tb.RowChunk(h, x_big[h:])], sketch_rows=64, seed=3)
    assert rel_err(parts.factor.entries, whole.factor.entries) <= 1e-12
    assert rel_err(parts.sketch.entries, whole.sketch.entries) <= 1e-12
    np.testing.assert_allclose(parts.stats.l1, whole.stats.l1, rtol=1e-12)
    assert parts.rows == whole.rows == m and parts.chunks == 2 and whole.chunks == 1


def test_fullsize_sketch_linearity(x_big):
    m = x_big.shape[0]
    h = m // 3
    s_all = dv.sketch(x_big, 0, 9, 128).cpu().numpy()
    s_a = dv.sketch(x_big[:h], 0, 9, 128).cpu().numpy()
    s_b = dv.sketch(x_big[h:], h, 9, 128).cpu().numpy()
    assert rel_err(s_a + s_b, s_all) <= 1e-12
    s2 = dv.sketch(x_big[:h] * 2.0, 0, 9, 128).cpu().numpy()
    assert np.array_equal(s2, 2.0 * s_a)


def test_fullsize_narrow_c4_shape():
    """C4 width (n = 25, warp-chain leaf + warp-pair tree) at 2^26 rows: R^T R = X^T X against the
    device Gram, stats agreement, split invariance."""
    m = 1 << 26
    spec = synthetic.config("C4", m=m)
    x = synthetic.generate(spec)
    r, l1, sq = dv.tsqr(x)
    g, gl1, _ = dv.gram(x)
    rn, gn = r.cpu().numpy(), g.cpu().numpy()
    assert np.array_equal(np.tril(rn, -1), np.zeros_like(rn)) and (np.diagonal(rn) >= 0).all()
    assert rel_err(rn.T @ rn, gn) <= 1e-10
    np.testing.assert_allclose(l1.cpu().numpy(), gl1.cpu().numpy(), rtol=1e-12)
    np.testing.assert_allclose(sq.cpu().numpy(), np.diagonal(gn), rtol=1e-12)
    h = m // 3 + 7
    r1, _, _ = dv.tsqr(x[:h])
    r2, _, _ = dv.tsqr(x[h:])
    both = tb.combine(tb.TriangularFactor(r1.cpu().numpy()), tb.TriangularFactor(r2.cpu().numpy()))
    assert rel_err(both.entries, rn) <= 1e-12
    del x
    torch.cuda.empty_cache()
