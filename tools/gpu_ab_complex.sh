#!/bin/bash
# A/B of the complex path: tools/old_libzz.so (previous build) vs the tree's library,
# alternating runs on one box
TAG=${1:-r02aj}
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2003_04776_b200 import _build; _build.build()"
timeout 600 python -m pytest tests/test_gpu_complex.py -m gpu -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_complex.log 2>&1; echo "pytest complex exit $?"; tail -1 $OUT/${TAG}_pytest_complex.log
for R in 1 2; do
for M in 4000 10000; do
  for V in "old 1" "new 1" "new 2" "new 4"; do
    set -- $V
    LIB=""; [ $1 = old ] && LIB="--lib tools/old_libzz.so"
    timeout 300 python tools/bench_complex.py --m $M --fusion $2 --no-check $LIB > $OUT/${TAG}_c.json 2> /dev/null
    python -c "import json; d=json.load(open('$OUT/${TAG}_c.json')); print('round $R m=$M $1 fusion $2', round(d['seconds_per_call']*1e3,2), 'ms')"
  done
done
done
