#!/bin/bash
# Iteration run on the GPU: smoke, fast GPU tests, diag kernel comparison, C3 and C4 bench.
TAG=${1:-it}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > $OUT/${TAG}_pytest.log 2>&1; echo "pytest exit $?"
tail -5 $OUT/${TAG}_pytest.log
timeout 900 python tools/cmp_diag.py > $OUT/${TAG}_cmp.log 2>&1; echo "cmp exit $?"
cat $OUT/${TAG}_cmp.log
timeout 600 python bench.py --config C3 --no-e2e --no-cpu > $OUT/${TAG}_bench_c3.json 2>$OUT/${TAG}_bench_c3.err; echo "c3 exit $?"
cat $OUT/${TAG}_bench_c3.json
timeout 900 python bench.py --no-e2e > $OUT/${TAG}_bench_c4.json 2>$OUT/${TAG}_bench_c4.err; echo "c4 exit $?"
cat $OUT/${TAG}_bench_c4.json
