#!/bin/bash
# A/B of the C5 training step: backward/train parity tests on the current build, then per
# variant library the CUPTI kernel table and the C5 bench value.
O=gpurun_out/abt
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_train.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for lib in paper_2503_14171_b200/libsplat_b200.so paper_2503_14171_b200/libsplat_b200_v*.so; do
  echo "== $lib"
  SPLAT_B200_LIB=$PWD/$lib timeout 300 python tools/kprof_train.py 4 3 2 2>&1 | grep -vi warn | head -14
  SPLAT_B200_LIB=$PWD/$lib timeout 300 python bench.py --workload train --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done 2>&1 | tee $O/kprof.txt
