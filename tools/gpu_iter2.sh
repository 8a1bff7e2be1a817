#!/bin/bash
# build, GPU tests (fast subset or all), per-config sweep, C4 bench (device only)
TAG=${1:-r02l}
TESTS=${2:-"tests/test_gpu.py"}
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2003_04776_b200 import _build; _build.build()"
timeout 1500 python -m pytest $TESTS -m gpu -x -q -p no:cacheprovider > $OUT/${TAG}_pytest.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/${TAG}_pytest.log
timeout 900 python tools/sweep.py > $OUT/${TAG}_sweep.json 2> $OUT/${TAG}_sweep.err; echo "sweep exit $?"
python - <<PY
import json
d=json.load(open("$OUT/${TAG}_sweep.json"))
def walk(x, p=''):
    if isinstance(x, dict):
        if 'median_ms' in x and 'config' in x: print(x['config'], x.get('mb'), round(x['median_ms'],3), 'ms', round(x.get('tflops',0),2), 'TF')
        for k,v in x.items(): walk(v, p+'/'+k)
    elif isinstance(x, list):
        for v in x: walk(v, p)
walk(d)
PY
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench exit $?"
python -c "import json; d=json.loads(open('$OUT/${TAG}_bench.json').read()); print('C4', d['ms_per_step'], d['value'], d.get('roofline',{}).get('frac'))"
