#!/bin/bash
# A/B: committed build vs variants/bk32 (BK = 32, 2 stages); the variant's library is copied
# over the in-tree one on the GPU box for the second half
OUT=gpurun_out
for v in base bk32; do
  if [ $v = bk32 ]; then cp variants/bk32/paper_2003_04776_b200/libzz.so paper_2003_04776_b200/libzz.so; fi
  timeout 200 python -m pytest tests/test_gpu.py -m gpu -x -q -p no:cacheprovider -k "C1 or C2_parity" > $OUT/bk_${v}_pytest.log 2>&1; echo "pytest $v $?"; tail -1 $OUT/bk_${v}_pytest.log
  for c in C4 C3; do
    timeout 250 python bench.py --config $c --steps 2 --warmup 2 --no-e2e --no-cpu > $OUT/bk_${v}_$c.json 2>&1
    tail -1 $OUT/bk_${v}_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', 'TF %.2f ms %.1f upd %.2f TF (%.3f ms) share %.3f' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['avg_launch_ms'], d['roofline']['share_of_step']))" 2>&1 | tail -1
  done
done
