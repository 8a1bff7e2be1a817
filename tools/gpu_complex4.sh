#!/bin/bash
TAG=${1:-r02e}
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2003_04776_b200 import _build; _build.build()"
for LA in 0 1; do for M in 4000 10000; do
  timeout 600 python tools/bench_complex.py --m $M --lookahead $LA --no-check > $OUT/${TAG}_complex_${M}_la$LA.json 2> $OUT/${TAG}_complex_${M}_la$LA.err; echo "bench $M la$LA exit $?"
  tail -1 $OUT/${TAG}_complex_${M}_la$LA.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('m', d['m'], 'la', d['lookahead'], 'ms %.2f TF %.2f' % (d['seconds_per_call']*1e3, d['value']))"
done; done
CMD="python tools/bench_complex.py --m 10000 --steps 1 --warmup 0 --no-check --lookahead 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zupdate -s 30 -c 1 -o $OUT/${TAG}_zupdate $CMD > $OUT/${TAG}_ncu_zupdate.log 2>&1; echo "ncu zupdate exit $?"
