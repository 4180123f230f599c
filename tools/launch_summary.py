"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0][:70]
    v = float(r[vi].replace(',', ''))
    v *= {'nsecond': 1, 'usecond': 1e3, 'msecond': 1e6, 'second': 1e9}.get(r[ui], 1)
    agg[name][0] += 1; agg[name][1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'total us':>10} {'n':>5} {'share':>6} {'us/launch':>10}  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{t/1e3:10.1f} {n:5d} {100*t/tot:5.1f}% {t/1e3/n:10.2f}  {k}")
