#!/bin/bash
# complex path A/B: builds of libzz (paper_2003_04776_b200/libzz*.so listed in LIBS) x step-group
# length, alternating runs on one box; then the launch list and k_zupdate captures
TAG=${1:-r02ak}
LIBS=${LIBS:-"libzz.so"}
MS=${MS:-"4000 10000"}
FS=${FS:-"2 3 4"}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_complex.py -m gpu -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_complex.log 2>&1; echo "pytest complex exit $?"; tail -1 $OUT/${TAG}_pytest_complex.log
P=paper_2003_04776_b200
for R in 1 2; do
for M in $MS; do
  for L in $LIBS; do
  for F in $FS; do
    timeout 300 python tools/bench_complex.py --m $M --fusion $F --no-check --lib $P/$L > $OUT/${TAG}_c.json 2> /dev/null
    python -c "import json; d=json.load(open('$OUT/${TAG}_c.json')); print('round $R m=$M $L fusion $F', round(d['seconds_per_call']*1e3,2), 'ms')"
  done
  done
done
done
if [ "${NCU:-1}" = "1" ]; then
CMD="python tools/bench_complex.py --m 10000 --steps 1 --warmup 0 --no-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_complex_launches.csv $CMD > /dev/null 2>&1; echo "ncu launches exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zupdate -s 100 -c 5 -o $OUT/${TAG}_zupdate $CMD > /dev/null 2>&1; echo "ncu zupdate exit $?"
fi
