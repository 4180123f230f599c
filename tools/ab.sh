#!/bin/bash
# A/B: parity subset on the current build, then per-variant pipeline fps and CUPTI kernel times.
O=gpurun_out/ab
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider ${PYTEST_K} > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
VIEWS=64 bash tools/variants.sh 2>&1 | tee $O/variants.txt
for lib in paper_2503_14171_b200/libsplat_b200.so paper_2503_14171_b200/libsplat_b200_v*.so; do
  echo "== $lib"; SPLAT_B200_LIB=$PWD/$lib timeout 300 python tools/kprof.py ${CFG:-c3} 10 2>&1 | grep -E "raster|fill|preproc|total|upscale|fixup"
done | tee $O/kprof.txt
