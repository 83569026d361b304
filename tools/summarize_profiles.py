"""Turn gpurun_out/ ncu artefacts of tools/gpu_round.sh into text summaries under profiles/ (round tag argv[1])."""
import collections, csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out_dir = os.environ.get("TSNMF_PROFILE_OUT") or os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)
g = os.path.join(ROOT, "gpurun_out")

def launches():
    rows = list(csv.reader(open(os.path.join(g, "launches.csv"))))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]; ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[ix["Metric Value"]].replace(",", ""))
        v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ix["Metric Unit"]], 1)
        name = r[ix["Kernel Name"]].split("(")[0]
        agg[name][0] += 1; agg[name][1] += v
    tot = sum(v for _, v in agg.values())
    lines = [f"# ncu launch list ({tag}): python bench.py --rows 4194304 --steps 2 --warmup 1 --no-cpu --no-e2e",
             "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)",
             f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}"]
    for name, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name[:60]:60s} {n:8d} {v / 1e6:10.3f} {100 * v / tot:6.2f}%")
    open(os.path.join(out_dir, f"{tag}_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
    subprocess.run(["cp", os.path.join(g, "launches.csv"), os.path.join(out_dir, f"{tag}_launches.csv")])

def full(rep, name, desc):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines())); d = dict(zip(r[0], r[2])); u = dict(zip(r[0], r[1]))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size"] + \
           [k for k in r[0] if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    lines = [f"# ncu --set full ({tag}): {desc}"]
    for k in keys:
        if k in d and d[k] not in ("", "0"):
            lines.append(f"{k} = {d[k]} {u.get(k, '')}")
    open(os.path.join(out_dir, f"{tag}_{name}_ncu_full.txt"), "w").write("\n".join(lines) + "\n")

if len(sys.argv) > 2 and sys.argv[2] == "--one":  # summarize_profiles.py TAG --one REP NAME DESC
    full(sys.argv[3], sys.argv[4], sys.argv[5])
    print(open(os.path.join(out_dir, f"{tag}_{sys.argv[4]}_ncu_full.txt")).read())
    sys.exit(0)
if os.path.exists(os.path.join(g, "launches.csv")):
    launches()
for rep, name, desc in [("tsqr_leaf_full.ncu-rep", "tsqr_leaf", "tsqr_leaf_kernel on 2^21 x 200 (tools/run_kernel.py tsqr 2097152 200 1)"),
                        ("gram_full2.ncu-rep", "gram", "gram_kernel on 2^22 x 200 (tools/run_kernel.py gram 4194304 200 1)"),
                        ("skgemm_full.ncu-rep", "sketch_gemm", "sketch_gemm_kernel on 2^20 x 200, k=400"),
                        ("tsqr_warp_leaf_full.ncu-rep", "tsqr_warp_leaf",
                         "tsqr_warp_leaf_kernel<25,3> on 2^22 x 25 (C4 width; tools/run_kernel.py tsqr 4194304 25 1)"),
                        ("tsqr_small_full.ncu-rep", "tsqr_small_leaf",
                         "tsqr_small_leaf_kernel<28> on 2^22 x 25 (C4 width; tools/run_kernel.py tsqr 4194304 25 1)")]:
    if os.path.exists(os.path.join(g, rep)):
        full(os.path.join(g, rep), name, desc)
b = os.path.join(g, "bench_full.log")
if os.path.exists(b):
    line = [l for l in open(b) if l.startswith("{")][-1]
    open(os.path.join(out_dir, f"{tag}_bench_full.json"), "w").write(line)
print(sorted(os.listdir(out_dir)))
