#!/bin/bash
# Iteration run on the GPU (every command under its own timeout): fast GPU tests, diagonal
# solve comparison, C3 and C4 bench lines.
TAG=${1:-it}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > $OUT/${TAG}_pytest.log 2>&1; echo "pytest exit $?"
tail -4 $OUT/${TAG}_pytest.log
timeout 400 python tools/cmp_diag.py > $OUT/${TAG}_cmp.log 2>&1; echo "cmp exit $?"
cat $OUT/${TAG}_cmp.log
for c in C3 C4; do
  timeout 400 python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/${TAG}_$c.json 2>$OUT/${TAG}_$c.err; echo "$c exit $?"
  tail -1 $OUT/${TAG}_$c.json | cut -c1-1400
done
