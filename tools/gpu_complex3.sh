#!/bin/bash
# complex path with the own 3M update kernel: parity, timing, launch list, ncu of k_zupdate
TAG=${1:-r02d}
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2003_04776_b200 import _build; _build.build()"
timeout 600 python -m pytest tests/test_gpu_complex.py -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_complex.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/${TAG}_pytest_complex.log
for M in 4000 10000; do
  timeout 600 python tools/bench_complex.py --m $M > $OUT/${TAG}_complex_${M}.json 2> $OUT/${TAG}_complex_${M}.err; echo "bench $M exit $?"
  tail -1 $OUT/${TAG}_complex_${M}.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('m', d['m'], 'ms %.2f TF %.2f' % (d['seconds_per_call']*1e3, d['value']), d['parity_sample']['max_abs'])"
done
CMD="python tools/bench_complex.py --m 10000 --steps 1 --warmup 0 --no-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_complex_launches.csv $CMD > $OUT/${TAG}_complex_ncu.log 2>&1; echo "ncu launches exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zupdate -s 60 -c 1 -o $OUT/${TAG}_zupdate $CMD > $OUT/${TAG}_ncu_zupdate.log 2>&1; echo "ncu zupdate exit $?"
