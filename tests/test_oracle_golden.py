"""Pin the oracle (CPU restatement) against golden vectors produced by the live
reference (tests/golden/make_golden.py).  CPU only."""

import importlib.util
import os

import numpy as np
import pytest

from conftest import ROOT, SMALL_CASES, rel_err


def test_derive_stream_exact(golden_rng, oracle):
    for (seed, tag), want in zip(golden_rng["seeds_tags"], golden_rng["streams"]):
        assert oracle.derive_stream(int(seed), int(tag)) == int(want)
    assert oracle.derive_stream(0, 0) == 0x48218226FF3CD4BF


@pytest.mark.parametrize("impl", ["c", "numpy"])
def test_blocks_match_reference(golden_rng, oracle, impl):
    ub = oracle.uniform_block if impl == "c" else oracle.uniform_block_np
    nb = oracle.normal_block if impl == "c" else oracle.normal_block_np
    for i, (s, start, cnt) in enumerate(golden_rng["blocks"]):
        s, start, cnt = int(s), int(start), int(cnt)
        assert np.array_equal(ub(s, start, cnt), golden_rng[f"uniform_{i}"])
        np.testing.assert_allclose(nb(s, start % 2**63, cnt), golden_rng[f"normal_{i}"], rtol=1e-12, atol=1e-13)


def test_oracle_c_library_built(oracle):
    assert oracle._clib() is not None, "oracle/liboracle_rng.so missing: run __graft_entry__.build()"


def test_gaussian_rows(golden_rng, oracle):
    np.testing.assert_allclose(oracle.gaussian_rows(5, 0, 10, 4), golden_rng["gaussian_rows_5_0_10_4"], rtol=1e-12,
                               atol=1e-13)
    np.testing.assert_allclose(oracle.gaussian_rows(3, 1000, 16, 9), golden_rng["gaussian_rows_3_1000_16_9"],
                               rtol=1e-12, atol=1e-13)


def test_known_answer():
    # reference gaussian_rows(0,0,2,4)[0]
    from oracle import tsnmf_oracle as o

    np.testing.assert_allclose(o.gaussian_rows(0, 0, 2, 4)[0], [-0.17660189, -1.602133, -0.92933372, 0.58165972],
                               atol=5e-8)


def test_reference_compiled_rng_if_built(golden_rng):
    """oracle/_ref holds the reference's own _kernels.c compiled (build container + GPU box)."""
    d = os.path.join(ROOT, "oracle", "_ref")
    so = [f for f in os.listdir(d) if f.startswith("_kernels")] if os.path.isdir(d) else []
    if not so:
        pytest.skip("reference RNG not built (no /root/reference here)")
    spec = importlib.util.spec_from_file_location("_kernels", os.path.join(d, so[0]))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    for i, (s, start, cnt) in enumerate(golden_rng["blocks"]):
        assert np.array_equal(mod.uniform_block(int(s), int(start), int(cnt)), golden_rng[f"uniform_{i}"])


@pytest.mark.parametrize("name", SMALL_CASES)
@pytest.mark.parametrize("size", [1, 7, 64, None])
@pytest.mark.parametrize("order", ["tree", "sequential", "first-come"])
def test_stream_pass_matches_reference(golden_tsqr, oracle, name, size, order):
    x = golden_tsqr[f"{name}__x"]
    size = x.shape[0] if size is None else size
    key = f"{name}__c{size}__{order}"
    res = oracle.stream_pass(oracle.chunks_of(x, size), sketch_rows=6, seed=11, combine_order=order)
    assert rel_err(res.r, golden_tsqr[key + "__r"]) <= 1e-14
    np.testing.assert_allclose(res.l1, golden_tsqr[key + "__l1"], rtol=1e-14)
    np.testing.assert_allclose(res.l2, golden_tsqr[key + "__l2"], rtol=1e-14)
    assert rel_err(res.sketch, golden_tsqr[key + "__sketch"]) <= 1e-13
    assert [res.rows, res.chunks, res.tree_depth] == list(golden_tsqr[key + "__meta"])


def test_spec_known_answers(golden_tsqr, oracle):
    np.testing.assert_allclose(oracle.factor_chunk(np.array([[3.0, 0], [4, 0], [0, 5]])), np.diag([5.0, 5.0]),
                               atol=1e-15)
    assert np.array_equal(oracle.factor_chunk(np.array([[1.0, 2, 2]])), golden_tsqr["fc_row"])
    assert np.array_equal(oracle.factor_chunk(np.array([[-1.0, 2, -2]])), golden_tsqr["fc_negrow"])
    np.testing.assert_allclose(oracle.factor_chunk(golden_tsqr["fc_wide_in"]), golden_tsqr["fc_wide"], atol=1e-14)
    np.testing.assert_allclose(oracle.combine(np.diag([3.0, 4]), np.diag([4.0, 3])), golden_tsqr["comb_diag"],
                               atol=1e-15)


def test_errors(oracle):
    with pytest.raises(oracle.OracleError) as e:
        oracle.stream_pass(iter([]))
    assert e.value.kind == "data"
    with pytest.raises(oracle.OracleError) as e:
        oracle.stream_pass(oracle.chunks_of(np.ones((3, 5)), 2))
    assert e.value.kind == "data" and "tall-and-skinny" in str(e.value)
    with pytest.raises(oracle.OracleError) as e:
        oracle.stream_pass(oracle.chunks_of(np.ones((9, 2)), 2), combine_order="bogus")
    assert e.value.kind == "usage"


def test_c1_generator_pinned(golden_c1, oracle):
    """The config generator feeding both sides is deterministic (checksums from
    the fixture run) and the reference recovered the planted set by SPA."""
    spec = oracle.config_spec("C1")
    mix, planted, perm = oracle.config_mixing(spec)
    assert np.array_equal(mix, golden_c1["mix"])
    assert list(planted) == list(golden_c1["planted"])
    x = oracle.config_rows(spec, 0, spec.m, mix)
    np.testing.assert_array_equal([x.sum(), (x * x).sum(), x[123, 45], x[9999, 199]], golden_c1["x_checksum"])
    assert sorted(golden_c1["k_spa"]) == sorted(golden_c1["planted"])


def test_c1_oracle_pass_matches_reference(golden_c1, oracle):
    spec = oracle.config_spec("C1")
    x = oracle.config_rows(spec, 0, spec.m)
    res = oracle.stream_pass(oracle.chunks_of(x, 8192), sketch_rows=120, seed=0)
    assert rel_err(res.r, golden_c1["r"]) <= 1e-14
    assert rel_err(res.sketch, golden_c1["sketch"]) <= 1e-13
    np.testing.assert_allclose(res.l1, golden_c1["l1"], rtol=1e-14)


def test_config_rows_are_row_addressed(oracle):
    """Any row range regenerates identically (counter addressing)."""
    for name in ("C1", "C4", "C5"):
        spec = oracle.config_spec(name, m=5000)
        mix = oracle.config_mixing(spec)[0]
        whole = oracle.config_rows(spec, 0, 300, mix)
        part = oracle.config_rows(spec, 100, 200, mix)
        assert np.array_equal(whole[100:300], part)
        assert (whole >= 0).all()


def test_oracle_selection_matches_reference(golden_select, oracle):
    """The oracle's SPA / XRAY / GP / NNLS restatement (select.py, nnls.py) reproduces the live
    reference's selections and coefficients (tests/golden/select.npz)."""
    for i in range(4):
        rr = golden_select[f"m{i}"]
        r = 4 if i < 2 else 8
        assert oracle.spa(rr, r, golden_select[f"m{i}_l1"]) == list(golden_select[f"m{i}_spa"])
        assert oracle.spa(rr, r) == list(golden_select[f"m{i}_spa_raw"])
        kx = oracle.xray_order(rr, r)
        assert kx == list(golden_select[f"m{i}_xray"])
        h = oracle.compute_h(rr, kx)
        np.testing.assert_allclose(h, golden_select[f"m{i}_h_xray"], atol=1e-12)
        assert abs(oracle.relative_residual(rr, kx, h) - golden_select[f"m{i}_res_xray"][0]) <= 1e-12
        gp, short = oracle.gp_select(golden_select[f"m{i}_sk"], r)
        assert gp == list(golden_select[f"m{i}_gp"]) and short == golden_select[f"m{i}_gp_short"][0]
    np.testing.assert_allclose(oracle.nnls_solve(golden_select["nnls_a"], golden_select["nnls_b"]),
                               golden_select["nnls_y"], atol=1e-13)


def test_oracle_c1_selection_matches_reference(golden_c1, oracle):
    red = oracle.reduced_matrix(golden_c1["r"])
    k_spa = oracle.spa(red, 20, golden_c1["l1"])
    assert k_spa == list(golden_c1["k_spa"])
    assert oracle.xray_order(red, 20) == list(golden_c1["k_xray"])
    h = oracle.compute_h(red, k_spa)
    np.testing.assert_allclose(h, golden_c1["h_spa"], atol=1e-10)
    sk = golden_c1["sketch"] / golden_c1["l1"]
    assert oracle.gp_select(sk, 20)[0] == list(golden_c1["k_gp"])


def test_oracle_nnls_iteration_cap_keeps_best_iterate(oracle):
    """nnls.py:96-103: hitting max_iter raises with the best iterate; best_effort keeps it."""
    rng = np.random.default_rng(3)
    a = rng.uniform(0, 1, (30, 6))
    b = a @ np.array([1.0, 0, 2, 0, 0.5, 0]) - 0.1 * rng.uniform(0, 1, 30)
    with pytest.raises(oracle.OracleNnlsIterationError) as e:
        oracle.nnls_solve(a, b, max_iter=1)
    assert e.value.best_y.shape == (6,) and (e.value.best_y >= 0).all()
    full = oracle.nnls_solve(a, b)
    assert (full >= 0).all()
