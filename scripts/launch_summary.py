"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; ki, mi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    agg[r[ki].split('(')[0]][0] += 1
    agg[r[ki].split('(')[0]][1] += float(r[mi].replace(',', '')) * scale[r[ui]]
tot = sum(v[1] for v in agg.values())
out = ["kernel,launches,total_us,share,avg_us"]
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(f'"{k}",{c},{t:.1f},{t / tot:.4f},{t / c:.2f}')
print("\n".join(out))
