"""Parity at the BASELINE configs' own row counts — TEST INFRASTRUCTURE (imports the oracle).

VERDICT r1 item 1: compare the device pass (TSQR R, column stats, GX sketch, Gram) and the reduced-space
selection / coefficients with the oracle's restatement of the reference (tsqr.py:276-343,
sketch.py:62-84, select.py:61-178, nnls.py:47-205) on the SAME X at the configs' full m:

  C2   2^26 x 200, k=400    TSQR + Gram + GX -> SPA, XRAY, GP, H
  C3   2^26 x 200, sigma=1e-2                  TSQR -> SPA, XRAY, H
  C5   2^28 x 64,  k=128    TSQR + Gram + GX -> XRAY, SPA, GP, H
  C4s  4e8 x 25 (one GPU's shard of C4 at g=4)  TSQR -> SPA, H

X is generated once on the device (synthetic.generate_into) and stays resident; the oracle side gets the
same bytes: X is copied device -> host block by block into anonymous shared memory and consumed by one
worker process per host core, each running the oracle's stream_pass (8192-row chunks, LAPACK QR per
chunk, reference TreeReducer) over a contiguous row range; the per-worker results are combined with the
reference's TreeReducer(combine) in row order (SURVEY §8d "best-effort CPU" order).

Criteria (north star + VERDICT r1): R normwise <= 1e-10, column l1/l2 and sketch <= 1e-12, Gram <= 1e-13,
selected K identical, H <= 1e-8 (max abs).

NNLS at the iteration cap.  At these m the reduced matrix's entries scale with sqrt(m) while the
reference's stationarity tolerance is an absolute 1e-8 (nnls.py:25,60-103), so some columns' Lawson-Hanson
iterations stall a hair above it and the reference raises NnlsIterationError (carrying ``best_y``).  Which
columns stall is decided by rounding, on either side.  The product's default mode keeps the reference's
contract (raise NumericalError("column i: ...") from NnlsIterationError; recorded as
``device_default_mode_error``); parity compares the iterates: both sides run in best-iterate mode (the
oracle's ``best_effort``, the device's ``capped=`` list — a capped column keeps its last iterate, exactly
the reference's ``best_y``), K from XRAY and H from compute_h must match, and the capped columns of each
side are listed.

    python tests/parity_full.py --configs C2,C3,C5,C4s --out profiles/r02_parity_full.json
    python tests/parity_full.py --scale 0.03125 ...      # reduced m (used by the -m gpu test)
"""

from __future__ import annotations

import argparse
import json
import mmap
import multiprocessing as mp
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CHUNK = 8192  # the reference's default RowChunk size (matio.py:27)
SLOT_BYTES = 65536 * 200 * 8  # one staging slot (105 MB); two per worker

# name -> (generator config, rows, sigma override, sketch k, gram, selections)
CASES = {
    "C2": ("C2", 1 << 26, None, 400, True, ("spa", "xray", "gp")),
    "C3": ("C3", 1 << 26, 1e-2, None, False, ("spa", "xray")),
    "C5": ("C5", 1 << 28, None, 128, True, ("xray", "spa", "gp")),
    "C4s": ("C4", 400_000_000, None, None, False, ("spa",)),
}

TOL = {"r": 1e-10, "stats": 1e-12, "sketch": 1e-12, "gram": 1e-13, "h": 1e-8}


# ---------------------------------------------------------------------------
# oracle workers (forked before CUDA is initialised in the parent)


def _worker(wid, q_in, q_out, bufs):
    try:
        from threadpoolctl import threadpool_limits

        from oracle import tsnmf_oracle as o

        while True:
            cfg = q_in.get()
            if cfg is None:
                return
            n, slot_rows = cfg["n"], cfg["slot_rows"]
            views = [np.ndarray((slot_rows, n), dtype=np.float64, buffer=b) for b in bufs]

            def chunks():
                while True:
                    msg = q_in.get()
                    if msg is None:
                        return
                    slot, off, rows = msg
                    blk = views[slot]
                    for c in range(0, rows, CHUNK):
                        yield off + c, blk[c:min(rows, c + CHUNK)]
                    # threads=1: the last chunk was reduced before the next item is requested
                    q_out.put(("free", wid, slot))

            t0 = time.perf_counter()
            with threadpool_limits(1):
                try:
                    res = o.stream_pass(chunks(), sketch_rows=cfg["k"], seed=cfg["seed"], with_gram=cfg["gram"])
                except o.OracleError as exc:
                    if "empty chunk stream" not in str(exc):
                        raise
                    q_out.put(("done", wid, {"rows": 0, "seconds": 0.0}))
                    continue
            q_out.put(("done", wid, {"r": res.r, "l1": res.l1, "sq": res.sumsq, "sketch": res.sketch,
                                     "gram": res.gram, "rows": res.rows, "chunks": res.chunks,
                                     "seconds": time.perf_counter() - t0}))
    except Exception:  # report, the parent raises
        q_out.put(("error", wid, traceback.format_exc()))


class OraclePool:
    def __init__(self, procs: int):
        ctx = mp.get_context("fork")
        self.procs = procs
        self.bufs = [[mmap.mmap(-1, SLOT_BYTES) for _ in range(2)] for _ in range(procs)]
        self.q_in = [ctx.Queue() for _ in range(procs)]
        self.q_out = ctx.Queue()
        self.ps = [ctx.Process(target=_worker, args=(w, self.q_in[w], self.q_out, self.bufs[w]), daemon=True)
                   for w in range(procs)]
        for p in self.ps:
            p.start()

    def run(self, x, k, seed, gram):
        """Stream the device matrix x through the workers; returns the combined oracle result."""
        import torch

        from oracle import tsnmf_oracle as o

        m, n = int(x.shape[0]), int(x.shape[1])
        slot_rows = (SLOT_BYTES // (8 * n)) // CHUNK * CHUNK
        views = [[torch.from_numpy(np.ndarray((slot_rows, n), dtype=np.float64, buffer=b)) for b in bw]
                 for bw in self.bufs]
        # contiguous row ranges, split at chunk boundaries
        bounds = [min(m, (w * m // self.procs) // CHUNK * CHUNK) for w in range(self.procs)] + [m]
        todo = [[(a, min(a + slot_rows, bounds[w + 1])) for a in range(bounds[w], bounds[w + 1], slot_rows)]
                for w in range(self.procs)]
        t0 = time.perf_counter()
        for w in range(self.procs):
            self.q_in[w].put({"n": n, "slot_rows": slot_rows, "k": k, "seed": seed, "gram": gram})

        sent_end = [False] * self.procs

        def feed(w, slot):
            a, b = todo[w].pop(0)
            views[w][slot][:b - a].copy_(x[a:b])
            self.q_in[w].put((slot, a, b - a))
            if not todo[w] and not sent_end[w]:  # FIFO: the end marker follows the last block
                self.q_in[w].put(None)
                sent_end[w] = True

        for w in range(self.procs):
            if not todo[w]:
                self.q_in[w].put(None)
                sent_end[w] = True
                continue
            feed(w, 0)
            if todo[w]:
                feed(w, 1)
        results = {}
        while len(results) < self.procs:
            kind, w, payload = self.q_out.get()
            if kind == "error":
                raise RuntimeError(f"oracle worker {w} failed:\n{payload}")
            if kind == "done":
                results[w] = payload
            elif todo[w]:
                feed(w, payload)
        parts = [results[w] for w in range(self.procs) if results[w]["rows"] > 0]

        def merge(a, b):
            return {"r": o.combine(a["r"], b["r"]), "l1": a["l1"] + b["l1"], "sq": a["sq"] + b["sq"],
                    "sketch": None if a["sketch"] is None else a["sketch"] + b["sketch"],
                    "gram": None if a["gram"] is None else a["gram"] + b["gram"],
                    "rows": a["rows"] + b["rows"], "chunks": a["chunks"] + b["chunks"]}

        red = o.TreeReducer(merge)
        for p in parts:
            red.push({k2: v for k2, v in p.items() if k2 != "seconds"})
        out = red.result()
        out["seconds"] = time.perf_counter() - t0
        out["worker_seconds_max"] = max(p["seconds"] for p in parts)
        return out

    def close(self):
        for q in self.q_in:
            q.put(None)
        for p in self.ps:
            p.join(timeout=10)


# ---------------------------------------------------------------------------
# comparisons


def rel(a, b) -> float:
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def maxrel(a, b) -> float:
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def spa_margins(mat: np.ndarray, r: int) -> float:
    """Smallest relative gap between the best and second-best SPA score over the r picks (tie risk)."""
    work = np.array(mat, dtype=np.float64, copy=True)
    taken = np.zeros(work.shape[1], dtype=bool)
    gaps = []
    for _ in range(r):
        sq = np.einsum("ij,ij->j", work, work)
        cand = np.where(taken, -np.inf, sq)
        order = np.argsort(cand)[::-1]
        j, j2 = int(order[0]), int(order[1])
        gaps.append(float((cand[j] - cand[j2]) / cand[j]) if np.isfinite(cand[j2]) else 1.0)
        taken[j] = True
        u = work[:, j].copy()
        work -= np.outer(u, u @ work) / (u @ u)
    return min(gaps)


def _attempt(fn):
    try:
        return fn(), None
    except Exception as exc:  # recorded, never raised: the reference itself may fail
        return None, f"{type(exc).__name__}: {exc}"


def run_case(label: str, pool: OraclePool, scale: float, seed: int = 0) -> dict:
    import torch

    import paper_1402_6964_b200 as tb
    from oracle import tsnmf_oracle as o
    from paper_1402_6964_b200 import synthetic

    cfg, rows, sigma, k, gram, sels = CASES[label]
    rows = max(CHUNK, int(rows * scale))
    over = {"seed": seed} if sigma is None else {"seed": seed, "sigma": sigma}
    spec = synthetic.config(cfg, **over)
    if rows > spec.m:
        spec = synthetic.config(cfg, m=rows, **over)
    # the generator is addressed by global row and m_total (C4s = the first 4e8 rows of C4's 1.6e9)
    n, r = spec.n, spec.r
    out = {"case": label, "config": cfg, "rows": rows, "n": n, "r": r, "k": k, "sigma": spec.sigma,
           "m_total_generator": spec.m, "full_size": rows == CASES[label][1], "bytes_x": rows * n * 8}
    x = torch.empty((rows, n), dtype=torch.float64, device="cuda")
    synthetic.generate_into(x, spec, 0)
    torch.cuda.synchronize()

    # --- device pass (the product, through the C ABI)
    t0 = time.perf_counter()
    res = tb.stream_pass([tb.RowChunk(0, x)], sketch_rows=k, seed=seed)
    g = tb.gram_pass([tb.RowChunk(0, x)]) if gram else None
    torch.cuda.synchronize()
    out["device_seconds"] = time.perf_counter() - t0

    # --- oracle pass on the same bytes
    ref = pool.run(x, k, seed, gram)
    out["oracle_seconds"] = ref["seconds"]
    out["oracle_procs"] = pool.procs
    out["oracle_chunks"] = ref["chunks"]
    del x
    torch.cuda.empty_cache()
    assert ref["rows"] == rows and res.rows == rows

    err = {"r": rel(res.factor.entries, ref["r"]),
           "l1": maxrel(res.stats.l1, ref["l1"]), "l2": maxrel(res.stats.l2, np.sqrt(ref["sq"]))}
    if k:
        err["sketch"] = rel(res.sketch.entries, ref["sketch"])
    if gram:
        err["gram"] = rel(g.gram, ref["gram"])
        err["gram_vs_RtR_oracle"] = rel(ref["r"].T @ ref["r"], ref["gram"])
    out["errors"] = err

    # --- reduced-space selection: product (device kernels where they exist) vs oracle on its own R
    red_dev = tb.rsvd(res.factor)
    red_ref = o.reduced_matrix(ref["r"])
    sel = {}
    h_cases = []
    if "spa" in sels:
        kd, e1 = _attempt(lambda: list(tb.spa(red_dev, r, normalize=True, stats=res.stats).indices))
        ko, e2 = _attempt(lambda: o.spa(red_ref, r, ref["l1"]))
        sel["spa"] = {"device": kd, "oracle": ko, "identical": kd == ko and kd is not None,
                      "device_error": e1, "oracle_error": e2,
                      "min_score_gap": spa_margins(red_ref / ref["l1"], r)}
        if kd is not None:
            h_cases.append(("spa", kd, ko))
    if "xray" in sels:
        from paper_1402_6964_b200.extremes import xray_order_device

        xcap: list = []
        kd, e1 = _attempt(lambda: xray_order_device(red_dev.reduced_matrix(), r, capped=xcap))
        kraise, eraise = _attempt(lambda: list(tb.xray_greedy(red_dev, r, device=True).indices))
        ko, e2 = _attempt(lambda: o.xray_order(red_ref, r, best_effort=True))
        kh, e3 = _attempt(lambda: list(tb.xray_greedy(red_dev, r).indices))
        sel["xray"] = {"device": kd, "oracle": ko, "identical": kd == ko and kd is not None,
                       "device_error": e1, "oracle_error": e2, "device_capped_refits": xcap,
                       "device_default_mode": kraise, "device_default_mode_error": eraise,
                       "product_host": kh, "product_host_error": e3}
        if kd is not None:
            h_cases.append(("xray", kd, ko))
    if "gp" in sels and k:
        kd = list(tb.gp_select(tb.scale_columns(res.sketch, res.stats), r).indices)
        ko = o.gp_select(ref["sketch"] / ref["l1"], r)[0]
        sel["gp"] = {"device": kd, "oracle": ko, "identical": kd == ko}
    for name, kd, ko in h_cases:
        from paper_1402_6964_b200.nonneg import solve_columns_device

        hcap: list = []
        mdev = red_dev.reduced_matrix()
        hd, e1 = _attempt(lambda: solve_columns_device(mdev[:, kd], mdev, capped=hcap))
        hor, e2 = _attempt(lambda: o.compute_h(red_ref, kd, best_effort=True))
        _, eraise = _attempt(lambda: tb.compute_h(red_dev, kd, device=True).entries)
        hh, e3 = _attempt(lambda: tb.compute_h(red_dev, kd).entries)
        d = {"device_error": e1, "oracle_error": e2, "product_host_error": e3,
             "device_default_mode_error": eraise}
        if hd is not None and hor is not None:
            d["max_abs_diff"] = float(np.abs(hd - hor[0]).max())
            d["capped_oracle_columns"] = hor[1]
            d["capped_device_columns"] = hcap
            d["within_tol"] = d["max_abs_diff"] <= TOL["h"]
            d["residual_device"] = float(tb.relative_residual(red_dev, kd, tb.CoefficientMatrix(hd, tuple(kd))))
            d["residual_oracle"] = o.relative_residual(red_ref, kd, hor[0])
        sel[f"h_{name}"] = d
    out["selection"] = sel
    # planted-set recovery (information only)
    planted = synthetic.mixing(spec)[1]
    out["planted"] = sorted(planted)

    ok = err["r"] <= TOL["r"] and err["l1"] <= TOL["stats"] and err["l2"] <= TOL["stats"]
    ok &= err.get("sketch", 0.0) <= TOL["sketch"] and err.get("gram", 0.0) <= TOL["gram"]
    ok &= all(v.get("identical", True) for key, v in sel.items() if not key.startswith("h_"))
    ok &= all(v.get("within_tol", False) for key, v in sel.items() if key.startswith("h_"))
    out["pass"] = bool(ok)
    out["tolerances"] = TOL
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3,C5,C4s")
    ap.add_argument("--scale", type=float, default=1.0, help="fraction of each config's m (1 = full)")
    ap.add_argument("--procs", type=int, default=0)
    ap.add_argument("--out", default="")
    args = ap.parse_args(argv)
    procs = args.procs or len(os.sched_getaffinity(0))
    pool = OraclePool(procs)  # forked before CUDA is initialised
    report = {"host_cores": len(os.sched_getaffinity(0)), "procs": procs, "scale": args.scale, "cases": []}
    try:
        with open("/proc/meminfo") as f:
            report["host_mem_gb"] = int(f.readline().split()[1]) / 1e6
    except OSError:
        pass
    try:
        for label in args.configs.split(","):
            t0 = time.perf_counter()
            case = run_case(label, pool, args.scale)
            case["wall_seconds"] = time.perf_counter() - t0
            report["cases"].append(case)
            print(json.dumps({kk: case[kk] for kk in ("case", "rows", "pass", "errors", "wall_seconds")}),
                  flush=True)
            if args.out:
                with open(args.out, "w") as f:
                    json.dump(report, f, indent=1, default=str)
    finally:
        pool.close()
    report["all_pass"] = all(c["pass"] for c in report["cases"])
    if args.out:
        with open(args.out, "w") as f:
            json.dump(report, f, indent=1, default=str)
    return report


if __name__ == "__main__":
    rep = main()
    print("ALL PASS" if rep["all_pass"] else "FAIL")
