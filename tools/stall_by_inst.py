"""Per-instruction-class stall breakdown from an ncu SASS source page CSV (ncu -i rep --page source --csv --print-source sass)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]].replace(',', ''))
    except Exception: return 0.0
kinds = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in data)
agg = collections.defaultdict(lambda: collections.Counter())
for r in data:
    op = r[ix['Source']].strip().split(' ')[0]
    if op.startswith('@'): op = r[ix['Source']].strip().split(' ')[1]
    op = op.split('.')[0]
    for k in kinds: agg[op][k] += f(r, k)
    agg[op]['all'] += f(r, 'Warp Stall Sampling (All Samples)')
print('total samples', tot)
for op, c in sorted(agg.items(), key=lambda kv: -kv[1]['all'])[:15]:
    top = ', '.join(f"{k[6:]} {100*v/tot:.1f}" for k, v in c.most_common(6) if k != 'all' and v > 0)
    print(f"{op:12s} {100*c['all']/tot:5.1f}%  {top}")
