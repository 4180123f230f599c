#!/bin/bash
# C5 training step time for each variant library in paper_2503_14171_b200/libsplat_b200_*.so
for lib in paper_2503_14171_b200/libsplat_b200.so paper_2503_14171_b200/libsplat_b200_*.so; do
  SPLAT_B200_LIB=$PWD/$lib timeout 300 python bench.py --workload train --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d.get('roofline') or {}
print('$lib'.split('/')[-1], 'view-steps/s', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'bwd ms/view', r.get('ms_per_view'))" || echo "$lib failed"
done
