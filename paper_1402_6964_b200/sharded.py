"""Row-sharded multi-GPU pass: one process per GPU, X split
into contiguous row ranges, each rank reduces its shard on its own GPU, then
ONE all-gather of a packed buffer [R | l1 | sumsq | sketch | gram] over NCCL
(NVLink/NVSwitch), after which every rank combines the gathered factors in
the reference's TreeReducer order over rank index (reference tsqr.py:201-234)
with the device combine kernel and sums the additive parts in rank order.
The result is replicated and identical on every rank (deterministic), and
equals a single-GPU pass up to round-off.

The exchange logic is backend-agnostic (it only needs torch.distributed and a
``combine_stack`` callable) so it is covered on CPU with gloo in tests; the
product path always uses the CUDA combine.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import device as dv


def shard_range(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced row range [lo, hi) of rank ``rank``."""
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class ShardPartials:
    """Per-rank reduction outputs (tensors on one device)."""

    r: object
    l1: object
    sumsq: object
    rows: int
    sketch: object = None
    gram: object = None


def _pack(p: ShardPartials, n: int, k: int):
    t = dv.torch()
    parts = ([] if p.r is None else [p.r.reshape(-1)]) + [p.l1.reshape(-1), p.sumsq.reshape(-1)]
    if k:
        parts.append(p.sketch.reshape(-1))
    if p.gram is not None:
        parts.append(p.gram.reshape(-1))
    parts.append(t.tensor([float(p.rows)], dtype=t.float64, device=p.l1.device))
    return t.cat(parts)


def exchange(p: ShardPartials, combine_stack, group=None) -> ShardPartials:
    """All-gather the packed partials and combine them deterministically.

    combine_stack(rs: world x n x n) -> n x n factor, in TreeReducer order.  ``p.r`` may be None (a Gram- or
    sketch-only pass): then only the additive parts are exchanged.
    """
    import torch.distributed as dist

    t = dv.torch()
    world = dist.get_world_size(group)
    n = int(p.l1.shape[0])
    k = int(p.sketch.shape[0]) if p.sketch is not None else 0
    flat = _pack(p, n, k)
    gathered = t.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
    dist.all_gather_into_tensor(gathered, flat, group=group)
    gathered = gathered.view(world, flat.numel())
    off = 0

    def take(count, shape):
        nonlocal off
        out = gathered[:, off:off + count].reshape((world,) + shape)
        off += count
        return out

    rs = take(n * n, (n, n)) if p.r is not None else None
    l1s = take(n, (n,))
    sqs = take(n, (n,))
    sks = take(k * n, (k, n)) if k else None
    gs = take(n * n, (n, n)) if p.gram is not None else None
    rows = take(1, (1,))

    def ordered_sum(stack):
        acc = stack[0].clone()
        for i in range(1, stack.shape[0]):
            acc = acc + stack[i]
        return acc

    r = combine_stack(rs.contiguous()) if rs is not None else None
    return ShardPartials(r=r, l1=ordered_sum(l1s), sumsq=ordered_sum(sqs), rows=int(rows.sum().item()),
                         sketch=ordered_sum(sks) if sks is not None else None,
                         gram=ordered_sum(gs) if gs is not None else None)


def reduce_shard(x_local, row_offset: int, *, sketch_rows: int | None = None, seed: int = 0,
                 with_gram: bool = False) -> ShardPartials:
    """This rank's device reduction of its resident shard."""
    r, l1, sq = dv.tsqr(x_local, stats=True)
    sk = dv.sketch(x_local, row_offset, seed, sketch_rows) if sketch_rows else None
    g = dv.gram(x_local, stats=False)[0] if with_gram else None
    return ShardPartials(r=r, l1=l1, sumsq=sq, rows=int(x_local.shape[0]), sketch=sk, gram=g)


def sharded_stream_pass(x_local, row_offset: int, *, sketch_rows: int | None = None, seed: int = 0,
                        with_gram: bool = False, group=None):
    """Multi-GPU ``stream_pass`` over a row-sharded, device-resident X.
    Returns (StreamResult, gram or None), replicated on every rank."""
    from .errors import DataError
    from .factor import ColumnStats, StreamResult, TriangularFactor
    from .projection import SketchResult

    local = reduce_shard(x_local, row_offset, sketch_rows=sketch_rows, seed=seed, with_gram=with_gram)
    out = exchange(local, dv.combine_factors, group=group)
    n = int(out.r.shape[0])
    if out.rows < n:
        raise DataError(f"not tall-and-skinny: m = {out.rows} < n = {n}")
    import torch.distributed as dist

    world = dist.get_world_size(group)
    stats = ColumnStats(l1=out.l1.cpu().numpy(), l2=np.sqrt(out.sumsq.cpu().numpy()))
    sk = SketchResult(entries=out.sketch.cpu().numpy(), seed=seed) if out.sketch is not None else None
    res = StreamResult(factor=TriangularFactor(entries=out.r.cpu().numpy()), stats=stats, sketch=sk,
                       rows=out.rows, chunks=world, tree_depth=world.bit_length())
    return res, (out.gram.cpu().numpy() if out.gram is not None else None)
