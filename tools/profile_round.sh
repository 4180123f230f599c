#!/bin/bash
# Round evidence on the GPU box: bench lines (no profiler), then the ncu launch
# list of a short bench command and one --set full capture per key kernel.
# Usage (via gpurun): bash tools/profile_round.sh  -> gpurun_out/prof/*
set -o pipefail
O=gpurun_out/prof
mkdir -p $O
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 rc=$?"
timeout 600 python bench.py --workload train --steps 5 --warmup 3 > $O/bench_c5_train.json 2> $O/bench_c5.err; echo "bench c5 rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
for c in c2 c4; do timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"; done
timeout 300 python tools/kprof.py c3 10 > $O/kprof_c3.txt 2>&1; timeout 300 python tools/kprof_train.py 4 3 2 > $O/kprof_c5.txt 2>&1
CMD="python bench.py --views 16 --kernel-views 16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > /dev/null 2>&1 && echo "short bench ok"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $O/launches.csv $CMD > /dev/null 2>&1; echo "launch list rc=$?"
for k in raster_fwd_kernel upscale_x4_kernel fill_rows_kernel preprocess_kernel fixup_kernel; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
        -o $O/ncu_$k $CMD > /dev/null 2>&1; echo "ncu $k rc=$?"
done
CMD4="python bench.py --config c4 --views 4 --kernel-views 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upscale_x2_kernel -s 3 -c 1 \
    -o $O/ncu_upscale_x2_kernel $CMD4 > /dev/null 2>&1; echo "ncu upscale_x2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"raster_bwd_kernel|ssim_stats|ssim_grad|upscale_bwd" -s 4 -c 4 \
    -o $O/ncu_train python tools/kprof_train.py 1 1 > /dev/null 2>&1; echo "ncu train rc=$?"
ls -la $O
