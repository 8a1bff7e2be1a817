#!/bin/bash
# complex path: serialised launch list and one ncu --set full capture of a fused k_zupdate
TAG=${1:-r02ak}
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2003_04776_b200 import _build; _build.build()"
timeout 300 python tools/bench_complex.py --m 10000 > $OUT/${TAG}_complex_10000.json 2> $OUT/${TAG}_complex.err; echo "bench exit $?"
python -c "import json; d=json.load(open('$OUT/${TAG}_complex_10000.json')); print('complex m=10000', round(d['seconds_per_call']*1e3,2), 'ms', round(d['value'],2), 'TF', d.get('parity_sample',{}).get('max_abs'))"
CMD="python tools/bench_complex.py --m 10000 --steps 1 --warmup 0 --no-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_complex_launches.csv $CMD > /dev/null 2>&1; echo "ncu launches exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zupdate -s 60 -c 1 -o $OUT/${TAG}_zupdate $CMD > /dev/null 2>&1; echo "ncu zupdate exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zdiag -s 60 -c 1 -o $OUT/${TAG}_zdiag $CMD > /dev/null 2>&1; echo "ncu zdiag exit $?"
