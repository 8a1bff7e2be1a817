#!/bin/bash
OUT=gpurun_out
for Z in 0 1; do
  ZZ_Z3M=$Z timeout 300 python -m pytest tests/test_gpu_complex.py -x -q -p no:cacheprovider > $OUT/z3m${Z}_pytest.log 2>&1; echo "pytest z3m$Z exit $?"; tail -1 $OUT/z3m${Z}_pytest.log
  for M in 4000 10000; do
    ZZ_Z3M=$Z timeout 300 python tools/bench_complex.py --m $M > $OUT/z3m${Z}_$M.json 2>&1
    tail -1 $OUT/z3m${Z}_$M.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('z3m$Z m', d['m'], 'ms %.2f TF %.2f' % (d['seconds_per_call']*1e3, d['value']), d['parity_sample']['max_abs'])"
  done
done
