#!/bin/bash
# Step grouping A/B: GPU tests of the modes, then C4 / C3 with ZZ_FUSE=2 and 3.
OUT=gpurun_out; TAG=${1:-f3}
timeout 600 python -m pytest tests/test_gpu.py -q -x -p no:cacheprovider -k "fusion or repeat or select or stress or sharded" > $OUT/${TAG}_pytest.log 2>&1; echo "pytest $?"; tail -4 $OUT/${TAG}_pytest.log
for cfg in C4 C3; do
for f in 2 3 2 3; do
  ZZ_FUSE=$f timeout 250 python bench.py --config $cfg --steps 2 --warmup 2 --no-e2e --no-cpu > $OUT/${TAG}_${cfg}_$f.json 2>&1
  tail -1 $OUT/${TAG}_${cfg}_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg fuse$f', 'TF %.2f ms %.1f upd %.2f TF (%.3f ms x %d) share %.3f' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['avg_launch_ms'], d['roofline']['update_launches_per_step'], d['roofline']['share_of_step']))" 2>&1 | tail -1
done
done
