"""Multi-rank exchange of the row-sharded pass (paper_1402_6964_b200.sharded)
on CPU with gloo, world_size 2: each rank reduces its shard (oracle as the
per-rank reducer — test infrastructure), the product's exchange() all-gathers
the packed partials and combines them in TreeReducer order; the replicated
result must equal the single-process oracle pass and be identical on both
ranks."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_combine_stack(rs):
    from oracle import tsnmf_oracle as o

    red = o.TreeReducer(o.combine)
    for r in rs.numpy():
        red.push(r)
    return torch.from_numpy(red.result())


def _worker(rank, world, port, x, k, seed, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import tsnmf_oracle as o
        from paper_1402_6964_b200 import sharded

        lo, hi = sharded.shard_range(x.shape[0], world, rank)
        xs = x[lo:hi]
        r = o.factor_chunk(xs)
        l1, sq = o.block_stats(xs)
        sk = o.sketch_block(xs, lo, k, seed)
        g = xs.T @ xs
        part = sharded.ShardPartials(r=torch.from_numpy(r), l1=torch.from_numpy(l1), sumsq=torch.from_numpy(sq),
                                     rows=hi - lo, sketch=torch.from_numpy(sk), gram=torch.from_numpy(g))
        out = sharded.exchange(part, _oracle_combine_stack)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), r=out.r.numpy(), l1=out.l1.numpy(),
                 sq=out.sumsq.numpy(), sk=out.sketch.numpy(), g=out.gram.numpy(), rows=out.rows)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_exchange_matches_single_pass(tmp_path, world, oracle):
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, (901, 13))
    k, seed = 5, 9
    mp.spawn(_worker, args=(world, _free_port(), x, k, seed, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for key in ("r", "l1", "sq", "sk", "g"):
        assert np.array_equal(outs[0][key], outs[1][key]), f"ranks disagree on {key}"
    ref = oracle.stream_pass(oracle.chunks_of(x, 451), sketch_rows=k, seed=seed)
    r = outs[0]
    assert np.linalg.norm(r["r"] - ref.r) / np.linalg.norm(ref.r) < 1e-13
    np.testing.assert_allclose(r["l1"], ref.l1, rtol=1e-13)
    np.testing.assert_allclose(r["sq"], ref.sumsq, rtol=1e-13)
    np.testing.assert_allclose(r["sk"], ref.sketch, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(r["g"], x.T @ x, rtol=1e-12)
    assert int(r["rows"]) == x.shape[0]


def _torch_r(x):
    """Sign-fixed R by torch (a CPU stand-in for the device leaf / combine kernels)."""
    r = torch.linalg.qr(x, mode="r")[1]
    n = x.shape[1]
    if r.shape[0] < n:
        r = torch.cat([r, torch.zeros(n - r.shape[0], n, dtype=r.dtype)])
    return r * torch.where(torch.diagonal(r) < 0, -1.0, 1.0).to(r.dtype)[:, None]


def _torch_combine_stack(rs):
    """The product's TreeReducer (factor.TreeReducer, reference tsqr.py:201-234) over rank index with a torch
    pair combine: the same order the device combine_factors uses."""
    from paper_1402_6964_b200.factor import TreeReducer

    red = TreeReducer(lambda a, b: _torch_r(torch.cat([a, b])))
    for r in rs:
        red.push(r)
    return red.result()


def _worker_torch(rank, world, port, x, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1402_6964_b200 import sharded

        lo, hi = sharded.shard_range(x.shape[0], world, rank)
        xs = torch.from_numpy(x[lo:hi])
        part = sharded.ShardPartials(r=_torch_r(xs), l1=xs.abs().sum(0), sumsq=(xs * xs).sum(0), rows=hi - lo,
                                     gram=xs.T @ xs)
        out = sharded.exchange(part, _torch_combine_stack)
        # Gram-only exchange (no factor packed; bench.py's Gram step at N > 1)
        gonly = sharded.exchange(sharded.ShardPartials(r=None, l1=part.l1, sumsq=part.sumsq, rows=hi - lo,
                                                       gram=part.gram), _torch_combine_stack)
        assert gonly.r is None and gonly.rows == out.rows
        np.savez(os.path.join(out_dir, f"t{world}_rank{rank}.npz"), r=out.r.numpy(), l1=out.l1.numpy(),
                 sq=out.sumsq.numpy(), g=out.gram.numpy(), rows=out.rows, has_sk=out.sketch is not None,
                 g_only=gonly.gram.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_product_packing_without_oracle(tmp_path, world, oracle):
    """exchange() with no sketch (packing without the optional block), a torch per-rank reduction and a torch
    pair combine in TreeReducer order (odd world = leftover subtree fold); the oracle only checks."""
    x = np.random.default_rng(11).standard_normal((777, 9))
    mp.spawn(_worker_torch, args=(world, _free_port(), x, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"t{world}_rank{r}.npz") for r in range(world)]
    for o in outs[1:]:
        for key in ("r", "l1", "sq", "g"):
            assert np.array_equal(outs[0][key], o[key]), f"ranks disagree on {key}"
    out = outs[0]
    assert not bool(out["has_sk"]) and int(out["rows"]) == x.shape[0]
    ref = oracle.stream_pass(oracle.chunks_of(x, 259), sketch_rows=None, seed=0)
    assert np.linalg.norm(out["r"] - ref.r) / np.linalg.norm(ref.r) < 1e-13
    assert np.all(np.diagonal(out["r"]) >= 0) and not np.tril(out["r"], -1).any()
    np.testing.assert_allclose(out["l1"], ref.l1, rtol=1e-13)
    np.testing.assert_allclose(out["sq"], ref.sumsq, rtol=1e-13)
    np.testing.assert_allclose(out["g"], x.T @ x, rtol=1e-12, atol=1e-12)
    assert np.array_equal(out["g_only"], out["g"])
