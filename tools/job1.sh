set -o pipefail
mkdir -p gpurun_out/j1
SPLAT_B200_LIB=$PWD/paper_2503_14171_b200/libsplat_b200_stats.so timeout 300 python tools/raster_stats.py c3 > gpurun_out/j1/stats_c3.txt 2>&1
SPLAT_B200_LIB=$PWD/paper_2503_14171_b200/libsplat_b200_stats.so timeout 300 python tools/raster_stats.py c5 > gpurun_out/j1/stats_c5.txt 2>&1
rm paper_2503_14171_b200/libsplat_b200_stats.so
CMD="python bench.py --views 16 --kernel-views 16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:raster_fwd_kernel -s 3 -c 1 -o gpurun_out/j1/rf $CMD > gpurun_out/j1/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/j1/rf.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/j1/rf_source.csv 2>&1
ls -la gpurun_out/j1
