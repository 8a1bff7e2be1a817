#!/bin/bash
# complex step groups: GPU tests of the complex path, bench_complex over (fusion, lookahead),
# then the real path's (tile, fusion, lookahead) sweep
TAG=${1:-r02ah}
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2003_04776_b200 import _build; _build.build()"
timeout 900 python -m pytest tests/test_gpu_complex.py -m gpu -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_complex.log 2>&1; echo "pytest complex exit $?"; tail -3 $OUT/${TAG}_pytest_complex.log
for M in 4000 10000; do
  for FL in "1 1" "2 1" "3 1" "4 1" "4 0"; do
    set -- $FL
    timeout 300 python tools/bench_complex.py --m $M --fusion $1 --lookahead $2 $( [ $M = 4000 ] && echo --no-check ) > $OUT/${TAG}_complex_${M}_f$1_la$2.json 2> $OUT/${TAG}_complex_${M}_f$1_la$2.err
    python -c "import json; d=json.load(open('$OUT/${TAG}_complex_${M}_f$1_la$2.json')); print('complex m=$M fusion $1 la $2', round(d['seconds_per_call']*1e3,2), 'ms', round(d['value'],2), 'TF', d.get('parity_sample',{}).get('max_abs'))"
  done
done
if [ "${SWEEP:-1}" = "1" ]; then
timeout 1500 python tools/tile_fusion_sweep.py C2 C3 C4 > $OUT/${TAG}_tf.json 2> $OUT/${TAG}_tf.err; echo "tf sweep exit $?"
cat $OUT/${TAG}_tf.err | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config'], d['mb'], d['fusion'], d['lookahead'], round(d['median_ms'], 3), d['bitwise_vs_first_of_tile'])"
fi
