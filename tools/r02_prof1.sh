#!/bin/bash
O=gpurun_out/prof1
mkdir -p $O
SPLAT_B200_LIB=$PWD/paper_2503_14171_b200/libsplat_b200_STATS.so timeout 300 python tools/raster_stats.py c3 > $O/raster_stats_c3.txt 2>&1
rm -f paper_2503_14171_b200/libsplat_b200_STATS.so
VIEWS=64 bash tools/variants.sh > $O/variants.txt 2>&1
CMD="python bench.py --views 16 --kernel-views 16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > /dev/null 2>&1 && echo "short bench ok"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:raster_fwd_kernel -s 3 -c 1 \
    -o $O/ncu_raster_fwd $CMD > $O/ncu.log 2>&1; echo "ncu rc=$?"
