#!/bin/bash
# The GPU test suite against the checked build (SPLAT_DCHECK bounds / ring-protocol
# checks compiled in) -- the stand-in for compute-sanitizer, which is closed on this pool.
O=gpurun_out/checked
mkdir -p $O
SPLAT_B200_LIB=$PWD/paper_2503_14171_b200/libsplat_b200_checked.so python -c "
from paper_2503_14171_b200 import _lib; assert _lib.load().splat_build_checked() == 1; print('checked build loaded')"
SPLAT_B200_LIB=$PWD/paper_2503_14171_b200/libsplat_b200_checked.so timeout 1500 \
  python -m pytest tests -m gpu -q -p no:cacheprovider -k "not multiprocess" > $O/gputest_checked.log 2>&1
echo "checked suite rc=$?"; tail -3 $O/gputest_checked.log; grep -c "SPLAT_DCHECK failed" $O/gputest_checked.log
SPLAT_B200_LIB=$PWD/paper_2503_14171_b200/libsplat_b200_checked.so timeout 900 python tools/sanitize.py > $O/sanitize_checked.log 2>&1; echo "sanitize.py (checked) rc=$?"; tail -2 $O/sanitize_checked.log
