"""Per-launch table (time, DRAM and L2 bytes) from an ncu --csv metrics dump (dev aid)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mn, mv, mu, ii = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= mv:
        continue
    d.setdefault((r[ii], r[ki].split('(')[0]), {})[r[mn]] = (float(r[mv].replace(',', '')), r[mu])
TS = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3}
BS = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'B': 1, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}
tot = 0.0
for (i, k), m in d.items():
    t = m['gpu__time_duration.sum']
    tus = t[0] * TS[t[1]]
    mb = lambda x: x[0] * BS[x[1]] / 1e6
    rd, wr = mb(m['dram__bytes_read.sum']), mb(m['dram__bytes_write.sum'])
    l2 = mb(m['lts__t_bytes.sum']) if 'lts__t_bytes.sum' in m else float('nan')
    tot += tus
    print(f"{i:>4} {k[:30]:30s} {tus:8.1f} us  dram r {rd:7.1f} w {wr:7.1f} MB  L2 {l2:8.1f} MB  "
          f"-> {(rd + wr) / tus:5.2f} TB/s")
print(f"total {tot:.1f} us")
