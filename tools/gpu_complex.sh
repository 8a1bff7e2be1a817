#!/bin/bash
# complex-pencil path: GPU tests, timing at m = 4000 / 10000, launch list and one ncu capture
TAG=${1:-r01j}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_complex.py -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_complex.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/${TAG}_pytest_complex.log
for M in 4000 10000; do
  timeout 600 python tools/bench_complex.py --m $M > $OUT/${TAG}_complex_$M.json 2> $OUT/${TAG}_complex_$M.err; echo "bench $M exit $?"; tail -1 $OUT/${TAG}_complex_$M.json; tail -3 $OUT/${TAG}_complex_$M.err
done
CMD="python tools/bench_complex.py --m 10000 --steps 1 --warmup 0 --no-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_complex_launches.csv $CMD > $OUT/${TAG}_complex_ncu.log 2>&1; echo "ncu launches exit $?"
