#!/bin/bash
OUT=gpurun_out; TAG=${1:-fu}
timeout 300 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > $OUT/${TAG}_pytest.log 2>&1; echo "pytest $?"; tail -3 $OUT/${TAG}_pytest.log
timeout 400 python -m pytest tests/test_gpu.py -m gpu -x -q -p no:cacheprovider -k "C5 or C3_full" > $OUT/${TAG}_pytest_slow.log 2>&1; echo "slow $?"; tail -3 $OUT/${TAG}_pytest_slow.log
for cfg in C4 C3; do
for f in 1 2 3; do
  ZZ_FUSE=$f timeout 250 python bench.py --config $cfg --steps 2 --warmup 2 --no-e2e --no-cpu > $OUT/${TAG}_${cfg}_$f.json 2>&1
  tail -1 $OUT/${TAG}_${cfg}_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg fuse$f', 'TF %.2f ms %.1f upd %.2f TF (%.3f ms x %d) share %.3f parity %s' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['avg_launch_ms'], d['roofline']['update_launches_per_step'], d['roofline']['share_of_step'], d.get('parity_sample')))" 2>&1 | tail -1
done
done
