"""Summarise an ncu SASS source page CSV: hottest instructions and shared-memory conflicts."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]].replace(',', ''))
    except Exception: return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print("total samples", tot)
top = sorted(range(len(data)), key=lambda i: -f(data[i], "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for i in sorted(top):
    r = data[i]
    print(f"{i:5d} {100*f(r,'Warp Stall Sampling (All Samples)')/tot:5.1f}% exc={f(r,'L1 Wavefronts Shared Excessive'):12.0f} {r[ix['Source']].strip()[:70]}")
print("--- top excessive shared wavefronts")
for i in sorted(range(len(data)), key=lambda i: -f(data[i], "L1 Wavefronts Shared Excessive"))[:12]:
    r = data[i]
    print(f"{i:5d} exc={f(r,'L1 Wavefronts Shared Excessive'):12.0f} ideal={f(r,'L1 Wavefronts Shared Ideal'):12.0f} {r[ix['Source']].strip()[:70]}")
