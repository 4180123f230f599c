"""Mean per-kernel metrics of an ncu --csv launch list (stdout mixed in is skipped)."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    lines = open(f).read().splitlines()
    i = next(k for k, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(lines[i:]))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    d = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        if len(r) == len(h):
            d[r[ki].split("(")[0][-28:]][r[mi]].append(float(r[vi].replace(",", "")))
    print(f)
    for k, m in d.items():
        n = len(m["gpu__time_duration.sum"])
        print(f"  {k:28s} n={n:3d}", {a.split("__")[1]: round(sum(v) / len(v) / (1e3 if "time" in a else 1e6), 2)
                                       for a, v in m.items()})
