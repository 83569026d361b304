"""Aggregate ncu SASS stall samples into regions split at BAR.SYNC / key markers."""
import csv, sys, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]].replace(',', ''))
    except Exception: return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
reg_start, acc, kinds = 0, 0.0, {}
def flush(end):
    global acc, kinds
    if acc / tot > 0.01:
        print(f"[{reg_start:5d}-{end:5d}] {100*acc/tot:5.1f}%  " + " ".join(f"{k}:{v}" for k, v in sorted(kinds.items(), key=lambda t: -t[1])[:6]))
    acc, kinds = 0.0, {}
for i, r in enumerate(data):
    src = r[ix['Source']].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
    acc += f(r, "Warp Stall Sampling (All Samples)")
    kinds[op.split('.')[0]] = kinds.get(op.split('.')[0], 0) + 1
    if op.startswith("BAR.SYNC") or op.startswith("WARPSYNC") and False:
        flush(i); reg_start = i + 1
flush(len(data) - 1)
