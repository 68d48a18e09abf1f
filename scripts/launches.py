"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui, ii = (hdr.index(k) for k in ('Kernel Name', 'Metric Value', 'Metric Unit', 'ID'))
mi = hdr.index('Metric Name') if 'Metric Name' in hdr else None
scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
for r in data:
    if len(r) <= vi or (mi is not None and r[mi] != 'gpu__time_duration.sum'):
        continue
    v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    name = r[ki].split('(')[0].replace('(anonymous namespace)::', '')[:48]
    agg[name][0] += 1
    agg[name][1] += v
    seq.append((int(r[ii]), name, v))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = sum(a[1] for a in agg.values())
print(f"{len(seq)} launches, {tot:.1f} us total")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{k:48s} n={n:4d} total={t:9.1f}us avg={t / n:8.2f}us share={t / tot:.3f}")
