#!/bin/bash
# time the raster stage for each variant library in paper_2503_14171_b200/libsplat_b200_v*.so
for lib in paper_2503_14171_b200/libsplat_b200.so paper_2503_14171_b200/libsplat_b200_v*.so; do
  SPLAT_B200_LIB=$PWD/$lib timeout 300 python bench.py --views ${VIEWS:-64} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], 'fps', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['stage_ms_per_view'].items()})" || echo "$lib failed"
done
