#!/bin/bash
# complex path on the final tree (tests, timings), then the full-size parity runs
TAG=${1:-r02an}
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2003_04776_b200 import _build; _build.build()"
timeout 600 python -m pytest tests/test_gpu_complex.py -m gpu -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_complex.log 2>&1; echo "pytest complex exit $?"; tail -1 $OUT/${TAG}_pytest_complex.log
for M in 2000 4000 10000; do
  timeout 600 python tools/bench_complex.py --m $M > $OUT/${TAG}_complex_$M.json 2> /dev/null
  python -c "import json; d=json.load(open('$OUT/${TAG}_complex_$M.json')); print('complex m=$M', round(d['seconds_per_call']*1e3,2), 'ms', round(d['value'],2), 'TF nominal', d.get('parity_sample',{}).get('max_abs'))"
done
timeout 600 python tools/full_parity.py --config C2 --chunks 4 --out $OUT/${TAG}_full_parity_c2.json 2> $OUT/${TAG}_fp_c2.err | tail -c 600; echo
timeout 4000 python tools/full_parity.py --config C4 --chunks 40 --budget ${BUDGET:-2700} --out $OUT/${TAG}_full_parity_c4.json 2> $OUT/${TAG}_fp_c4.err | tail -c 900; echo; tail -3 $OUT/${TAG}_fp_c4.err
