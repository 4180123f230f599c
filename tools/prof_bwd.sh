#!/bin/bash
# C5 backward kernels: launch durations (ncu, serialised) for the current build and the
# v* variant libraries, plus one --set full capture of each backward kernel of the build.
O=gpurun_out/pbwd
mkdir -p $O
K='regex:raster_bwd|reduce_pairs|chain_kernel'
for lib in paper_2503_14171_b200/libsplat_b200.so paper_2503_14171_b200/libsplat_b200_v*.so; do
  tag=$(basename $lib .so)
  SPLAT_B200_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -s 30 -c 30 --csv \
    python bench.py --workload train --steps 2 --warmup 3 --no-cpu-baseline --train-streams 1 > $O/launch_$tag.csv 2> $O/launch_$tag.err
  python - $O/launch_$tag.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; rows = rows[1:]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
d = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    d[r[ki][:40]][r[mi]].append(float(r[vi].replace(",", "")))
print(sys.argv[1])
for k, m in d.items():
    print(f"  {k:40s}", {n: round(sum(v) / len(v) / (1e3 if 'time' in n else 1e6), 2) for n, v in m.items()}, len(m['gpu__time_duration.sum']))
PY
done
for k in raster_bwd2_kernel reduce_pairs2_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 6 -c 1 -o $O/full_$k -f \
    python bench.py --workload train --steps 1 --warmup 3 --no-cpu-baseline --train-streams 1 > $O/full_$k.log 2>&1
  echo "$k rc=$?"
done
