#!/bin/bash
# quick GPU check: parity tests + short bench summary
set -o pipefail
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --views ${VIEWS:-128} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('fps', round(d['value'],1), 'stages', {k: round(v*1e3,1) for k,v in (d['stage_ms_per_view'] or {}).items()}, 'raster_frac', d['roofline'] and round(d['roofline']['frac'],3), 'up_frac', d['roofline_upscale'] and round(d['roofline_upscale']['frac'],3))"
