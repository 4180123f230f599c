#!/bin/bash
# ncu --set full of one raster_fwd_kernel launch (C3 bench views) -> gpurun_out/prof/
O=gpurun_out/prof
mkdir -p $O
CMD="python bench.py --views 16 --kernel-views 16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
timeout 600 $CMD > /dev/null 2>&1 && echo "short bench ok"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-raster_fwd_kernel} -s 3 -c 1 \
    -o $O/ncu_${TAG:-raster} $CMD > $O/ncu_${TAG:-raster}.log 2>&1; echo "ncu rc=$?"
