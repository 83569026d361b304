"""Benchmark of the single-pass reduction (BASELINE.json metric: 1-pass TSQR/Gram
GB/s of X and % of roofline), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--rows M]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
  python bench.py --impl reference            # the reference's CPU path (baseline/_ref, else the oracle port)

A step = one TSQR pass over the job's X (BASELINE config C2 by default: m = 2^26 rows, n = 200, fp64,
107 GB resident in HBM; X row-sharded evenly over the N GPUs = config C3, strong scaling), i.e. the
leaf kernel + on-GPU combine tree (+ for N > 1 one NCCL all-gather of the factors and the ordered
device combine).  Gram and GX (k = 400) passes over the same X are timed the same way and reported
under "gram" / "sketch".  X (107 GB) is far larger than L2 (126 MB), so no L2 flush is needed.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.0  # measured DMMA peak, profiles/r01_peaks.json (no FP64 entry in MEASURED_PEAKS.json)
FP64_FMA_PEAK_TFLOPS = 34.2  # measured DFMA peak (same file): the narrow warp-leaf TSQR runs on the FMA pipe
TSQR_N200_CAPTURE = "r02_tsqr_split_leaf_ncu_full.txt"  # ncu --set full of the n = 200 (split) leaf, 2^21 rows
METRIC = "1-pass TSQR/Gram GB/s of X and % of HBM peak at 1/2/4/8 B200 vs CPU ref"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md"


def ncu_traffic_per_row(path: str, rows: int):
    """dram bytes per row of the profiled leaf launch (profiles/r01_tsqr_leaf_ncu_full.txt, ncu --set full)."""
    try:
        vals = {}
        for line in open(path):
            if "=" in line and not line.startswith("#"):
                k, v = line.split("=", 1)
                num, unit = v.split()[0], v.split()[1] if len(v.split()) > 1 else ""
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)
                vals[k.strip()] = float(num) * scale
        return (vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]) / rows
    except Exception:
        return None


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C2")
    p.add_argument("--rows", type=int, default=None, help="override total rows m")
    p.add_argument("--k", type=int, default=None, help="sketch rows for the GX pass (default: the config's, "
                                                         "k=128 for C5, 400 otherwise)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-extra", action="store_true", help="skip the Gram / GX passes")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 7:
                    rows.append(parts)
        except Exception:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port of the reference's stream_pass on host cores


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    """The unmodified reference package installed into baseline/_ref (tools/install_reference.sh)."""
    return os.path.isfile(os.path.join(REF_DIR, "tsnmf", "tsqr.py"))


def _cpu_worker(args):
    """One host process: the reference's stream_pass over 8192-row RowChunks (two pre-generated chunks cycled:
    the QR cost is data-independent).  impl "reference" = the installed reference package itself
    (baseline/_ref, compiled backend, threads=1); "port" = the oracle's restatement of it."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import tsnmf_oracle as o

    spec_name, n_chunks, chunk_rows, seed, sketch, start_at, impl, threads = args
    spec = o.config_spec(spec_name)
    mix = o.config_mixing(spec)[0]
    bufs = [o.config_rows(spec, i * chunk_rows, chunk_rows, mix) for i in range(2)]
    if impl == "reference":
        sys.path.insert(0, REF_DIR)
        import tsnmf

        def run():
            chunks = (tsnmf.RowChunk(row_offset=i * chunk_rows, data=bufs[i % 2]) for i in range(n_chunks))
            res = tsnmf.stream_pass(chunks, sketch_rows=sketch, seed=seed, threads=threads)
            return res.rows, np.asarray(res.factor.entries)
    else:
        def run():
            res = o.stream_pass(((i * chunk_rows, bufs[i % 2]) for i in range(n_chunks)), sketch_rows=sketch,
                                seed=seed)
            return res.rows, np.asarray(res.r)
    while start_at and time.time() < start_at:  # all workers start the timed pass together
        time.sleep(0.001)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        rows, r = run()
        dt = time.perf_counter() - t0
    return dt, rows, r


def cpu_reference(spec_name: str, n: int, seconds: float, sketch=None, impl: str | None = None):
    """Time the reference's CPU pass (per-8192-row-chunk LAPACK QR + TreeReducer, reference
    tsqr.py:276-343) with one process per host core on a bounded sample; the per-process factors are
    combined with the reference TreeReducer(combine) (SURVEY.md §8d best-effort CPU).  impl: "reference" (the
    installed reference, default when present) or "port" (the oracle restatement)."""
    import multiprocessing as mpc

    import numpy as np

    from oracle import tsnmf_oracle as o

    impl = impl or ("reference" if reference_available() else "port")
    cores = len(os.sched_getaffinity(0))
    chunk_rows = 8192
    # calibrate: chunks on one core
    probe = _cpu_worker((spec_name, 4, chunk_rows, 0, sketch, 0, impl, 1))[0] / 4
    per_proc = max(2, int(seconds / max(probe, 1e-3)))
    ctx = mpc.get_context("fork")
    with ctx.Pool(cores) as pool:
        outs = pool.map(_cpu_worker, [(spec_name, per_proc, chunk_rows, 0, sketch, time.time() + 3.0, impl, 1)]
                        * cores)
    t0 = time.perf_counter()
    if impl == "reference":
        sys.path.insert(0, REF_DIR)
        import tsnmf

        red = tsnmf.tsqr.TreeReducer(tsnmf.combine)
        for _, _, r in outs:
            red.push(tsnmf.TriangularFactor(entries=np.array(r)))
    else:
        red = o.TreeReducer(o.combine)
        for _, _, r in outs:
            red.push(r)
    red.result()
    wall = max(dt for dt, _, _ in outs) + (time.perf_counter() - t0)
    rows = sum(r for _, r, _ in outs)
    gbs = rows * n * 8 / wall / 1e9
    what = ("the installed reference package (baseline/_ref: tsnmf.stream_pass, compiled backend, threads=1) "
            if impl == "reference" else "the oracle port of the reference's stream_pass ")
    return {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "reference" if impl == "reference" else "port",
            "sample": f"{rows} rows x {n} cols of {spec_name}: {cores} processes x {per_proc} chunks of "
                      f"{chunk_rows} rows, each running {what}(numpy/OpenBLAS LAPACK QR per chunk, 1 BLAS "
                      f"thread), factors combined by the reference TreeReducer(combine); time = slowest "
                      f"process + final combine" + (f"; + GX k={sketch}" if sketch else ""),
            "seconds": wall}


def as_shipped_reference(spec_name: str, n: int, seconds: float):
    """The reference as a user runs it: ONE process, tsnmf.stream_pass(chunks, threads=<cores>) (its
    thread-pool map, tsqr.py:247-273,315-333), 8192-row chunks, 1 BLAS thread."""
    import multiprocessing as mpc

    if not reference_available():
        return None
    cores = len(os.sched_getaffinity(0))
    probe = _cpu_worker((spec_name, 4, 8192, 0, None, 0, "reference", 1))[0] / 4
    n_chunks = max(8, int(seconds / max(probe, 1e-3)))
    ctx = mpc.get_context("fork")
    with ctx.Pool(1) as pool:
        dt, rows, _ = pool.apply(_cpu_worker, ((spec_name, n_chunks, 8192, 0, None, 0, "reference", cores),))
    return {"value": rows * n * 8 / dt / 1e9, "unit": "GB/s", "cores": cores, "kind": "reference",
            "sample": f"{rows} rows x {n} cols of {spec_name}: one process, tsnmf.stream_pass(threads={cores}) "
                      f"over 8192-row RowChunks (baseline/_ref, compiled backend, 1 BLAS thread)"}


def run_reference(args):
    """--impl reference: the reference's CPU path on the box's host cores (rank 0 only), best-effort form (one
    process per core); the as-shipped single-process number is printed beside it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import tsnmf_oracle as o

    spec = o.config_spec(args.config)
    steps = []
    base = None
    for _ in range(args.warmup + args.steps):
        base = cpu_reference(args.config, spec.n, max(2.0, args.cpu_seconds / 4))
        steps.append(base["value"])
    vals = steps[args.warmup:] or steps
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": base["seconds"] * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{args.config}: TSQR pass, m={spec.m}, n={spec.n} (bounded CPU sample)"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": base["cores"], "kind": base["kind"],
                             "sample": base["sample"]},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    try:
        shipped = as_shipped_reference(args.config, spec.n, max(4.0, args.cpu_seconds / 2))
        if shipped:
            line["as_shipped"] = shipped
    except Exception as exc:
        line["as_shipped"] = {"error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm



def selection_timing(x, r, n):
    """XRAY (r picks) + compute_h on the reduced matrix of x's R: device kernels vs the host code (the
    reference algorithm).  Each side may legitimately fail (e.g. the Lawson-Hanson iteration limit when
    it cycles at the tolerance); failures are reported, never raised."""
    import numpy as np
    import torch

    import paper_1402_6964_b200 as tb
    from paper_1402_6964_b200 import device as dv, extremes as ex, nonneg as nn

    r_mat, _, _ = dv.tsqr(x)
    mat = ex.as_matrix(tb.rsvd(tb.TriangularFactor(np.triu(r_mat.cpu().numpy()))))

    def attempt(fn, reps):
        try:
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                out = fn()
            torch.cuda.synchronize()
            return (time.perf_counter() - t0) * 1e3 / reps, out, None
        except Exception as exc:
            return None, None, f"{type(exc).__name__}: {exc}"

    sel = {"workload": f"XRAY r={r} + compute_h on the {n}x{n} reduced matrix of this pass",
           "host": "numpy/OpenBLAS Lawson-Hanson (reference algorithm), 1 process"}
    xd_ms, kd, err = attempt(lambda: ex.xray_order_device(mat, r), 3)
    sel.update(xray_device_ms=xd_ms, xray_device_error=err)
    xh_ms, kh, err = attempt(lambda: ex.xray_order(mat, r), 1)
    sel.update(xray_host_ms=xh_ms, xray_host_error=err)
    if kd is not None and kh is not None:
        sel["k_identical"] = list(kd) == list(kh)
    kset = kd if kd is not None else kh
    if kset is not None:
        hd_ms, hd, err = attempt(lambda: nn.solve_columns(mat[:, kset], mat, device=True), 3)
        sel.update(compute_h_device_ms=hd_ms, compute_h_device_error=err)
        hh_ms, hh, err = attempt(lambda: nn.solve_columns(mat[:, kset], mat), 1)
        sel.update(compute_h_host_ms=hh_ms, compute_h_host_error=err)
        if hd is not None and hh is not None:
            sel["h_max_abs_diff"] = float(np.abs(hd - hh).max())
    return {k: v for k, v in sel.items() if v is not None}

def e2e_legs(tb, x, n, devc):
    """Two more end-to-end legs through the public API (world 1): (a) the reference's default chunking —
    8192-row RowChunks from PAGEABLE host memory (matio.py:27; the host packs them into pinned staging);
    (b) a file in the reference's binary format through ChunkReader(device=...) with and without the
    reference's sha256 content hash (pipeline.py:157-159), the file already in the page cache."""
    import numpy as np
    import torch

    out = {}
    rows = min(int(x.shape[0]), 1 << 23)
    pool_rows = min(rows, (2 << 30) // (8 * n))
    pool = x[:pool_rows].cpu().numpy().copy()  # pageable

    def chunks():
        off = 0
        while off < rows:
            take = min(8192, rows - off)
            src = off % pool_rows
            take = min(take, pool_rows - src)
            yield tb.RowChunk(off, pool[src:src + take])
            off += take

    tb.stream_pass(chunks())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = tb.stream_pass(chunks())
    dt = time.perf_counter() - t0
    assert res.rows == rows
    out["pageable_8192"] = {"value": rows * n * 8 / dt / 1e9, "unit": "GB/s", "rows": rows,
                            "h2d_bytes_per_step": rows * n * 8, "d2h_bytes_per_step": (n * n + 2 * n) * 8,
                            "api": "stream_pass over 8192-row RowChunks of pageable numpy memory"}
    del pool
    frows = min(int(x.shape[0]), 1 << 21)
    fd, path = tempfile.mkstemp(suffix=".tsm")
    os.close(fd)
    try:
        tb.write_matrix(path, x[:frows].cpu().numpy())
        for label, hasher in (("file_device_reader", None), ("file_device_reader_sha256", "sha256")):
            best = None
            for _ in range(2):  # first read warms the page cache
                h = hashlib.sha256() if hasher else None
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = tb.stream_pass(tb.ChunkReader(path, device=devc, hasher=h))
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            assert res.rows == frows
            out[label] = {"value": frows * n * 8 / best / 1e9, "unit": "GB/s", "rows": frows,
                          "api": "stream_pass(ChunkReader(path, device=cuda" + (", hasher=sha256" if hasher else "")
                                 + ")), file in the page cache",
                          "bound": "host sha256 of the byte stream (sequential by definition)" if hasher
                                   else "page-cache read into pinned buffers"}
    finally:
        os.unlink(path)
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1402_6964_b200 as tb
    from paper_1402_6964_b200 import _native, sharded, synthetic
    from paper_1402_6964_b200 import device as dv

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    devc = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=devc)
    lib = _native.load()

    if args.k is None:
        args.k = 128 if args.config == "C5" else 400
    spec = synthetic.config(args.config)
    if args.rows:
        spec = synthetic.config(args.config, m=args.rows)
    m, n = spec.m, spec.n
    lo, hi = sharded.shard_range(m, world, rank)
    x = torch.empty((hi - lo, n), dtype=torch.float64, device=devc)
    mix = synthetic.mixing(spec)[0]
    synthetic.generate_into(x, spec, row0=lo, mix=mix)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=devc)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def tsqr_step():
        r, l1, sq = dv.tsqr(x, stats=True)
        if world > 1:
            part = sharded.ShardPartials(r=r, l1=l1, sumsq=sq, rows=hi - lo)
            sharded.exchange(part, dv.combine_factors)
        return r

    # N > 1: the product's exchange (sharded.exchange: one all-gather of the packed partials + ordered sum)
    def gram_step():
        g, l1, sq = dv.gram(x, stats=True)
        if world > 1:
            g = sharded.exchange(sharded.ShardPartials(r=None, l1=l1, sumsq=sq, rows=hi - lo, gram=g),
                                 dv.combine_factors).gram
        return g

    def sketch_step():
        s = dv.sketch(x, lo, 0, args.k)
        if world > 1:
            z = torch.zeros(n, dtype=torch.float64, device=devc)
            s = sharded.exchange(sharded.ShardPartials(r=None, l1=z, sumsq=z, rows=hi - lo, sketch=s),
                                 dv.combine_factors).sketch
        return s

    def timed(fn, steps, warmup, slot):
        for _ in range(warmup):
            fn()
        barrier()
        lib.tsnmf_profile_read(slot, None, None)  # drop warm-up events
        lib.tsnmf_profile_enable(1)
        launches0 = lib.tsnmf_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        barrier()
        lib.tsnmf_profile_enable(0)
        launches = lib.tsnmf_launch_count() - launches0
        ms = max_over_ranks(e0.elapsed_time(e1)) / steps
        tot = np.zeros(1)
        cnt = np.zeros(1, dtype=np.int64)
        import ctypes

        tms, tl = ctypes.c_double(), ctypes.c_longlong()
        _native.check(lib.tsnmf_profile_read(slot, ctypes.byref(tms), ctypes.byref(tl)))
        kern_ms = tms.value / max(tl.value, 1)
        del tot, cnt
        return ms, kern_ms, int(launches), int(tl.value)

    hbm, hbm_src = hbm_peak()
    bytes_total = m * n * 8
    bytes_local = (hi - lo) * n * 8
    with ClockSampler(local) as clk:
        ms, leaf_ms, launches, _ = timed(tsqr_step, args.steps, args.warmup, 0)
        # combine-tree share (same run, separate slot)
    clocks = clk.summary()
    value = bytes_total / (ms * 1e-3) / 1e9
    leaf_flops = 2.0 * n * n * (hi - lo)
    leaf_tf = leaf_flops / (leaf_ms * 1e-3) / 1e12
    plan = dv.tsqr_plan(n, hi - lo)
    narrow = plan["panel"] == 1  # n <= 32: register-block warp leaf (FP64 FMA), else the DMMA panel leaf
    # the committed ncu captures are per width: traffic is only reported for a width one was taken at
    captures = {25: ("r02_tsqr_warp_leaf_ncu_full.txt", 1 << 22), 64: ("r02_tsqr_reg_leaf_n64_ncu_full.txt", 1 << 21),
                200: (TSQR_N200_CAPTURE, 1 << 21)}
    prof_file, prof_rows = captures.get(n, ("(none)", 0))
    prof_n = n if n in captures else None
    tpr = ncu_traffic_per_row(os.path.join(ROOT, "profiles", prof_file), prof_rows) if prof_n else None
    peak_tf = FP64_FMA_PEAK_TFLOPS if narrow else FP64_PEAK_TFLOPS

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: TSQR pass (leaf + on-GPU combine tree"
                               f"{' + NCCL all-gather + ordered combine' if world > 1 else ''}), R + column l1/l2",
                   "m": m, "n": n, "r": spec.r, "sigma": spec.sigma, "rows_per_gpu": hi - lo,
                   "resident_gb_per_gpu": round(bytes_local / 1e9, 2), "parallelism": f"rows{world}",
                   "l2": "inputs (>=13 GB per GPU) exceed the 126 MB L2; no flush needed",
                   "tsqr_plan": plan},
        "roofline": {"bound": "tensor", "achieved": leaf_tf, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": leaf_tf / peak_tf,
                     "traffic": tpr * (hi - lo) if tpr else None,
                     "traffic_source": (f"ncu --set full dram__bytes_read+write of the leaf at m={prof_rows}, "
                                        f"n={prof_n} (profiles/{prof_file}), per row x rows per launch; "
                                        f"algorithmic {8 * n * (hi - lo)} B") if tpr else
                                       f"no committed ncu capture at n={n}",
                     "kernel": ("tsqr_warp_leaf_kernel (FP64 FMA, one Householder chain per warp)" if narrow
                                else "tsqr_split_leaf_kernel (FP64 DMMA m8n8k4; 256-row blocks, right column "
                                     "tiles in an L2 workspace)" if plan["block_rows"] == 256
                                else "tsqr_reg_leaf_kernel (one Householder chain per warp, row block in registers, "
                                     "FP64 DMMA m8n8k4 trailing updates)" if 28 <= n <= 64 and plan["ctas_per_sm"] == 1
                                else "tsqr_leaf_kernel (FP64 DMMA m8n8k4)"),
                     "algorithmic": f"2 n^2 = {2 * n * n} flop per row x {hi - lo} rows per launch",
                     "peak_source": ("measured FP64 DFMA peak" if narrow else "measured FP64 DMMA peak")
                                    + ", profiles/r01_peaks.json",
                     "kernel_ms": leaf_ms, "share_of_step": leaf_ms / ms,
                     "hbm_gbs": bytes_local / (leaf_ms * 1e-3) / 1e9,
                     "hbm_frac": bytes_local / (leaf_ms * 1e-3) / 1e9 / hbm, "hbm_peak": hbm,
                     "hbm_peak_source": hbm_src},
        "gpu_launches": launches,
        "clocks": clocks,
    }

    if not args.no_extra:
        gms, gk_ms, _, _ = timed(gram_step, max(2, args.steps), 1, 2)
        gflops = 1.0 * n * (n + 1) * (hi - lo)
        line["gram"] = {"value": bytes_total / (gms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": gms,
                        "kernel_ms": gk_ms, "kernel_tflops": gflops / (gk_ms * 1e-3) / 1e12,
                        "frac_fp64": gflops / (gk_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                        "hbm_frac": bytes_local / (gk_ms * 1e-3) / 1e9 / hbm,
                        "kernel": ("gram_narrow_kernel (fragments from global memory, upper triangle in each warp's "
                                   "registers)" if n <= 64 else
                                   "gram_cyclic_kernel (25 tile columns, every tile pair once, accumulators in "
                                   "registers)" if 193 <= n <= 200 else "gram_kernel (staged, 16x16 super-tiles)"),
                        "ncu": {25: "profiles/r02_gram_narrow_n25_ncu_full.txt",
                                64: "profiles/r02_gram_narrow_n64_ncu_full.txt",
                                200: "profiles/r02_gram_cyclic_ncu_full.txt"}.get(n)}
        # size-independent full-m checks of this pass (parity against the oracle at full m is
        # tests/parity_full.py -> profiles/r02_parity_full.json): R^T R = X^T X with X^T X from
        # the independent Gram kernel, R upper triangular with a nonnegative diagonal
        r_full = tsqr_step() if world == 1 else None
        if r_full is not None:
            g_full = gram_step()
            rtr = r_full.T @ r_full
            line["checks"] = {
                "rtr_vs_gram_rel": float(torch.linalg.norm(rtr - g_full) / torch.linalg.norm(g_full)),
                "r_strict_lower_zero": bool((torch.tril(r_full, -1) == 0).all()),
                "r_diag_nonneg": bool((torch.diagonal(r_full) >= 0).all()),
                "tolerance": "rtr_vs_gram_rel <= 1e-10"}
        sms, sk_ms, _, _ = timed(sketch_step, 2, 1, 3)
        sflops = 2.0 * args.k * n * (hi - lo)
        line["sketch"] = {"value": bytes_total / (sms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": sms,
                          "k": args.k, "kernel_ms": sk_ms, "kernel_tflops": sflops / (sk_ms * 1e-3) / 1e12,
                          "frac_fp64_gemm_only": sflops / (sk_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                          "normals_per_s": args.k * (hi - lo) / (sk_ms * 1e-3)}

        # device selection + coefficients (§8f row 1) on this pass's reduced matrix vs the host code
        if rank == 0:
            try:
                line["selection"] = selection_timing(x, spec.r, n)
            except Exception as exc:  # never lose the headline line to an optional extra
                line["selection"] = {"error": f"{type(exc).__name__}: {exc}"}

    # end to end through the public API from pinned host buffers (H2D inside the timed region)
    if not args.no_e2e:
        pool_rows = min(hi - lo, (4 << 30) // (8 * n))
        host = torch.empty((pool_rows, n), dtype=torch.float64).pin_memory()
        host.copy_(x[:pool_rows].cpu())
        hnp = host.numpy()
        chunk_rows = 1 << 16

        def chunks():
            off = lo
            while off < hi:
                take = min(chunk_rows, hi - off)
                src = (off - lo) % pool_rows
                take = min(take, pool_rows - src)
                yield tb.RowChunk(off, hnp[src:src + take])
                off += take

        def e2e_step():
            res = tb.stream_pass(chunks())
            if world > 1:  # same exchange as the resident path: all-gather + ordered device combine
                part = sharded.ShardPartials(
                    r=torch.as_tensor(res.factor.entries, device=devc),
                    l1=torch.as_tensor(res.stats.l1, device=devc),
                    sumsq=torch.as_tensor(res.stats.l2 ** 2, device=devc), rows=res.rows)
                out = sharded.exchange(part, dv.combine_factors)
                out.r.cpu()
            return res

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        e_steps = 2
        for _ in range(e_steps):
            res = e2e_step()
        barrier()
        e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / e_steps)
        line["e2e"] = {"value": bytes_total / (e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e_ms,
                       "h2d_bytes_per_step": bytes_local, "d2h_bytes_per_step": (n * n + 2 * n) * 8,
                       "api": "paper_1402_6964_b200.stream_pass over host RowChunks (65536 rows each)"
                              + (" + NCCL all-gather + ordered device combine" if world > 1 else ""),
                       "host_pool": f"{pool_rows} pinned rows cycled (QR cost is data-independent)",
                       "steps": e_steps, "timer": "host wall clock around the API call, barrier on both sides"}
        assert res.rows == hi - lo
        if world == 1:
            line["e2e_legs"] = e2e_legs(tb, x, n, devc)

    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_reference(args.config, n, args.cpu_seconds)
            line["cpu_baseline"].pop("seconds", None)
        except Exception as exc:
            line["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
