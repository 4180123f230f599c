#!/bin/bash
# Round-2 profile evidence on one GPU (never under a multi-rank command):
#  * launch list (gpu__time_duration per launch) of a short C3 bench command
#  * ncu --set full of the key kernels (C3 views; C4 eye for x2; C5 training step)
#  * the upscalers in steady state (--cache-control none, 20th launch of the
#    4-buffer rotation, so the previous frames' write-back is in the window)
O=gpurun_out/prof2
mkdir -p $O
CMD="python bench.py --views 16 --kernel-views 16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
timeout 600 $CMD > $O/short_bench.json 2>&1 && echo "short bench ok"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv $CMD > /dev/null 2>&1; echo "launch list rc=$?"
for k in raster_fwd_kernel fixup_kernel preprocess_kernel fill_rows_kernel count_rows_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/ncu_$k $CMD > /dev/null 2>&1; echo "ncu $k rc=$?"
done
UP="python tools/upscale_bench.py"
timeout 900 ncu --set full --clock-control none --cache-control none -k regex:upscale_x4_kernel -s 20 -c 1 -o $O/ncu_upscale_x4_steady $UP > /dev/null 2>&1; echo "ncu x4 rc=$?"
timeout 900 ncu --set full --clock-control none --cache-control none -k regex:upscale_x2_kernel -s 20 -c 1 -o $O/ncu_upscale_x2_steady $UP > /dev/null 2>&1; echo "ncu x2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"raster_bwd_kernel|ssim_stats|ssim_grad|upscale_bwd|reduce_pairs|raster_fwd_kernel" -s 12 -c 6 \
    -o $O/ncu_train python tools/kprof_train.py 1 1 1 > /dev/null 2>&1; echo "ncu train rc=$?"
ls -la $O
