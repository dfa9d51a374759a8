"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel count, total ms, share."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(',', ''))
    except ValueError:
        continue
    scale = {'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0, 'nsecond': 1e-6}.get(r[ui], 1e-6)
    name = r[ki].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '')
    agg[name][0] += 1
    agg[name][1] += v * scale
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:70]:70s} {c:6d} {v:10.3f} ms {100 * v / tot:6.2f}%")
