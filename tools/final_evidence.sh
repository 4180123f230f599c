#!/bin/bash
# Round-end evidence: standalone bench lines for every config (no profiler), the launch list
# of a short C3 command, and ncu --set full captures of the kernels changed this round.
O=gpurun_out/final
mkdir -p $O
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --config c2 --no-extras > $O/bench_c2.json 2>/dev/null; echo "c2 rc=$?"
timeout 600 python bench.py --config c4 --no-extras > $O/bench_c4.json 2>/dev/null; echo "c4 rc=$?"
timeout 600 python bench.py --workload train --steps 5 --warmup 3 > $O/bench_c5.json 2>/dev/null; echo "c5 rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2>/dev/null; echo "ref rc=$?"
timeout 300 python tools/kprof.py c3 10 > $O/kprof_c3.txt 2>&1
timeout 300 python tools/kprof_train.py 4 3 1 > $O/kprof_c5_1stream.txt 2>&1
timeout 300 python tools/upscale_bench.py > $O/upscale_steady.txt 2>&1
CMD="python bench.py --views 16 --kernel-views 16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv $CMD > /dev/null 2>&1; echo "launch list rc=$?"
for k in raster_fwd_kernel fixup_kernel fill_rows_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/ncu_$k $CMD > /dev/null 2>&1; echo "ncu $k rc=$?"
done
for k in raster_bwd2_kernel reduce_pairs2_kernel ssim_stats_kernel ssim_grad_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 1 -o $O/ncu_$k \
    python bench.py --workload train --steps 1 --warmup 3 --no-cpu-baseline --train-streams 1 > /dev/null 2>&1; echo "ncu $k rc=$?"
done
