#!/bin/bash
# GPU box: full -m gpu suite, the three sanitizers on tools/sanitize.py, one bench line.
O=gpurun_out/r02
mkdir -p $O
rm -f gpurun_out/parity.jsonl
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/gputest.log 2>&1; echo "pytest rc=$?"
tail -5 $O/gputest.log
for t in ${SAN_TOOLS:-memcheck racecheck synccheck}; do
  timeout 900 compute-sanitizer --tool $t --print-limit 40 python tools/sanitize.py > $O/san_$t.log 2>&1; echo "$t rc=$?"
  tail -3 $O/san_$t.log
done
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
  cut -c1-400 $O/bench.json
fi
