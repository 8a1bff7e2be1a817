#!/bin/bash
OUT=gpurun_out; TAG=${1:-ab4}
ZZ_UPD=6 timeout 200 python -m pytest tests/test_gpu.py -m gpu -x -q -p no:cacheprovider -k "C1 or C2 or ragged or leading or host or stress" > $OUT/${TAG}_pytest5.log 2>&1; echo "pytest v6 exit $?"; tail -2 $OUT/${TAG}_pytest5.log
for cfg in C4 C3; do
for v in 2 6; do
  ZZ_UPD=$v timeout 250 python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/${TAG}_${cfg}_$v.json 2>&1
  tail -1 $OUT/${TAG}_${cfg}_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg v$v', 'TF %.2f ms %.1f upd %.2f TF (%.3f ms) share %.3f' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['avg_launch_ms'], d['roofline']['share_of_step']))" 2>&1 | tail -1
done
done
