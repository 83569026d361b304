"""Print the headline ncu metrics of a .ncu-rep (first kernel): duration, IPC, issue, stalls per issue."""
import csv, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, v = rows[0], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
d = dict(zip(h, v))
for k in want:
    if k in d:
        print(f"{k:70s} {d[k]}")
st = [(float(x), k) for k, x in d.items() if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")
      and x.replace(".", "", 1).isdigit()]
for x, k in sorted(st, reverse=True)[:10]:
    if x > 0.02:
        print(f"{k.replace('smsp__average_warps_issue_stalled_', 'stall_'):70s} {x:.3f}")
