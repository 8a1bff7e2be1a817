#!/bin/bash
TAG=${1:-r01l}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_complex.py -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_complex.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/${TAG}_pytest_complex.log
for LA in 0 1; do for M in 4000 10000; do
  ZZ_ZLOOKAHEAD=$LA timeout 600 python tools/bench_complex.py --m $M > $OUT/${TAG}_complex_${M}_la$LA.json 2> $OUT/${TAG}_complex_${M}_la$LA.err; echo "bench $M la$LA exit $?"
  tail -1 $OUT/${TAG}_complex_${M}_la$LA.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('m', d['m'], 'ms %.2f TF %.2f' % (d['seconds_per_call']*1e3, d['value']), d['parity_sample']['max_abs'])"
done; done
CMD="python tools/bench_complex.py --m 10000 --steps 1 --warmup 0 --no-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_complex_launches.csv $CMD > $OUT/${TAG}_complex_ncu.log 2>&1; echo "ncu launches exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zdiag -s 100 -c 1 -o $OUT/${TAG}_zdiag $CMD > $OUT/${TAG}_ncu_zdiag.log 2>&1; echo "ncu zdiag exit $?"
