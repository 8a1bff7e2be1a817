#!/bin/bash
# Generic step groups: bitwise vs the previous build (default 3), tests, C4/C3 for k = 3..6.
OUT=gpurun_out; TAG=${1:-fn}
timeout 600 python tools/ab_lib.py paper_2003_04776_b200/libzz_old.so paper_2003_04776_b200/libzz.so C2:128 C2@1:64 C3:128 C5:128
ZZ_FUSE=2 timeout 600 python tools/ab_lib.py paper_2003_04776_b200/libzz_old.so paper_2003_04776_b200/libzz.so C2:64 C3:128
timeout 900 python -m pytest tests/test_gpu.py -q -x -p no:cacheprovider -k "fusion or repeat or select or stress or sharded or host_path" > $OUT/${TAG}_pytest.log 2>&1; echo "pytest $?"; tail -3 $OUT/${TAG}_pytest.log
for cfg in C4 C3; do
for f in 3 4 5 6 3 4; do
  ZZ_FUSE=$f timeout 250 python bench.py --config $cfg --steps 2 --warmup 2 --no-e2e --no-cpu > $OUT/${TAG}_${cfg}_$f.json 2>&1
  tail -1 $OUT/${TAG}_${cfg}_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg fuse$f', 'TF %.2f ms %.1f upd %.2f TF share %.3f' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['share_of_step']))" 2>&1 | tail -1
done
done
