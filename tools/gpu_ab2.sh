#!/bin/bash
# correctness + A/B of the update kernel variants (development)
OUT=gpurun_out; TAG=${1:-ab2}
for v in 4 2; do
  ZZ_UPD=$v timeout 300 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_v$v.log 2>&1; echo "pytest v$v exit $?"; tail -2 $OUT/${TAG}_pytest_v$v.log
done
for cfg in C4 C3; do
for v in "1 0" "2 0" "2 2" "4 0" "4 1"; do
  set -- $v
  ZZ_UPD=$1 ZZ_UPD_PERSIST=$2 timeout 400 python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/${TAG}_${cfg}_$1_$2.json 2>&1
  tail -1 $OUT/${TAG}_${cfg}_$1_$2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg v$1 p$2', 'TF %.2f ms %.1f upd %.2f TF (%.3f ms) share %.3f' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['avg_launch_ms'], d['roofline']['share_of_step']))" 2>&1 | tail -1
done
done
