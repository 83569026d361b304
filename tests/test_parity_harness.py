"""The full-size parity harness (tests/parity_full.py) on CPU: its block streaming through forked oracle
workers and the row-ordered TreeReducer(combine) of their results reproduce a direct oracle pass."""

import numpy as np
import torch

from conftest import rel_err


def test_oracle_pool_matches_direct_pass(oracle):
    import parity_full as pf

    old = pf.SLOT_BYTES
    pf.SLOT_BYTES = 3 * pf.CHUNK * 30 * 8  # 3 chunks per slot: many blocks per worker
    try:
        pool = pf.OraclePool(3)
        try:
            rng = np.random.default_rng(1)
            x = rng.uniform(0, 1, (7 * pf.CHUNK * 3 + 1234, 30))
            got = pool.run(torch.from_numpy(x), 9, 4, True)
            got2 = pool.run(torch.from_numpy(x[:5000]), None, 0, False)  # workers 1, 2 get no rows
        finally:
            pool.close()
    finally:
        pf.SLOT_BYTES = old
    ref = oracle.stream_pass(oracle.chunks_of(x, pf.CHUNK), sketch_rows=9, seed=4, with_gram=True)
    assert got["rows"] == x.shape[0] and got["chunks"] == ref.chunks
    assert rel_err(got["r"], ref.r) <= 1e-14
    assert rel_err(got["sketch"], ref.sketch) <= 1e-14
    assert rel_err(got["gram"], ref.gram) <= 1e-15
    np.testing.assert_allclose(got["l1"], ref.l1, rtol=1e-14)
    ref2 = oracle.factor_chunk(x[:5000])
    assert got2["rows"] == 5000 and rel_err(got2["r"], ref2) <= 1e-14


def test_spa_margin_helper():
    import parity_full as pf

    # scores 9, 4, 1 -> gap 5/9; after deflating column 0: 4 vs 1 -> gap 3/4
    assert abs(pf.spa_margins(np.diag([3.0, 2.0, 1.0]), 2) - 5.0 / 9.0) < 1e-15
