#!/bin/bash
OUT=gpurun_out; TAG=${1:-ab3}
timeout 300 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > $OUT/${TAG}_pytest.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/${TAG}_pytest.log
ZZ_UPD=3 timeout 300 python -m pytest tests/test_gpu.py -m "gpu and not slow" -x -q -p no:cacheprovider -k "C1 or C2 or ragged or leading" > $OUT/${TAG}_pytest_v3.log 2>&1; echo "pytest v3 exit $?"; tail -2 $OUT/${TAG}_pytest_v3.log
for cfg in C4 C3; do
for v in 2 3; do
  ZZ_UPD=$v timeout 400 python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/${TAG}_${cfg}_$v.json 2>&1
  tail -1 $OUT/${TAG}_${cfg}_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg v$v', 'TF %.2f ms %.1f upd %.2f TF (%.3f ms) share %.3f' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['avg_launch_ms'], d['roofline']['share_of_step']))" 2>&1 | tail -1
done
done
for mb in 64 96 128; do
  timeout 300 python bench.py --config C2 --mb $mb --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/${TAG}_C2_$mb.json 2>&1
  tail -1 $OUT/${TAG}_C2_$mb.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 mb$mb', 'TF %.2f ms %.2f upd %.2f TF share %.3f' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['share_of_step']))" 2>&1 | tail -1
done
