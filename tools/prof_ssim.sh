#!/bin/bash
# ncu --set full of the C5 SSIM kernels (one launch each, single view stream).
O=gpurun_out/pssim
mkdir -p $O
for k in ssim_stats_kernel ssim_grad_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 6 -c 1 -o $O/full_$k -f \
    python bench.py --workload train --steps 1 --warmup 3 --no-cpu-baseline --train-streams 1 > $O/full_$k.log 2>&1
  echo "$k rc=$?"
done
