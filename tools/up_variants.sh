for lib in paper_2503_14171_b200/libsplat_b200.so paper_2503_14171_b200/libsplat_b200_*.so; do
  SPLAT_B200_LIB=$PWD/$lib timeout 300 python tools/upscale_bench.py 2>&1 | grep -v Warn
done
timeout 300 python tools/kprof.py c3 10 > gpurun_out/kprof_c3.txt 2>&1
