#!/bin/bash
TAG=${1:-r01o}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke exit $?"; tail -2 $OUT/${TAG}_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/${TAG}_pytest_gpu.log
for Z in 1 0; do for M in 4000 10000; do
  ZZ_Z3M=$Z timeout 300 python tools/bench_complex.py --m $M > $OUT/${TAG}_complex_${M}_z3m$Z.json 2>&1
  tail -1 $OUT/${TAG}_complex_${M}_z3m$Z.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('z3m$Z m', d['m'], 'ms %.2f TF %.2f' % (d['seconds_per_call']*1e3, d['value']), d['parity_sample']['max_abs'])"
done; done
CMD="python tools/bench_complex.py --m 10000 --steps 1 --warmup 0 --no-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_complex_launches.csv $CMD > $OUT/${TAG}_complex_ncu.log 2>&1; echo "ncu launches exit $?"
