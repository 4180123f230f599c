#!/bin/bash
# CUPTI per-kernel times (C3) for each variant library; $1 = kernel-name regex
for lib in paper_2503_14171_b200/libsplat_b200.so paper_2503_14171_b200/libsplat_b200_*.so; do
  echo "$lib"; SPLAT_B200_LIB=$PWD/$lib timeout 300 python tools/kprof.py ${CFG:-c3} 10 2>&1 | grep -E "$1"
done
