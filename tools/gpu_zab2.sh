#!/bin/bash
# k_zdiag columns-per-warp variants: bitwise A/B against the one-column kernel, complex tests on
# the tree's library, then timings (alternating)
TAG=${1:-r02am}
OUT=gpurun_out
mkdir -p $OUT
P=paper_2003_04776_b200
python tools/ab_zlib.py $P/libzz_old.so $P/libzz_c1w32.so $P/libzz_c2w16.so $P/libzz_c2w32.so $P/libzz_c4w16.so $P/libzz_c4w8.so 2>&1 | tee $OUT/${TAG}_bitwise.txt
timeout 600 python -m pytest tests/test_gpu_complex.py -m gpu -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_complex.log 2>&1; echo "pytest complex exit $?"; tail -1 $OUT/${TAG}_pytest_complex.log
for R in 1 2; do
for M in 2000 4000 10000; do
  for L in libzz_old.so libzz_c1w32.so libzz_c2w16.so libzz_c2w32.so libzz_c4w16.so libzz_c4w8.so; do
    timeout 300 python tools/bench_complex.py --m $M --no-check --lib $P/$L > $OUT/${TAG}_c.json 2> /dev/null
    python -c "import json; d=json.load(open('$OUT/${TAG}_c.json')); print('round $R m=$M $L', round(d['seconds_per_call']*1e3,2), 'ms')"
  done
done
done 2>&1 | tee $OUT/${TAG}_times.txt
