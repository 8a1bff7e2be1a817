#!/bin/bash
# k_update v1/v2 A/B at C4 and an ncu capture of k_diag3 mid-wavefront at C4 (development)
OUT=gpurun_out; TAG=${1:-pf}
for v in 1 2; do
  ZZ_UPD=$v timeout 400 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/${TAG}_upd$v.json 2>&1; echo "upd v$v exit $?"
  tail -1 $OUT/${TAG}_upd$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v', $v, 'TF %.2f ms %.1f upd %.2f TF (%.3f ms) share %.3f' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['avg_launch_ms'], d['roofline']['share_of_step']))"
done
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 400 $CMD > $OUT/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_diag3 -s 150 -c 1 -o $OUT/${TAG}_diag3 $CMD > $OUT/${TAG}_ncu_diag3.log 2>&1; echo "ncu diag3 $?"
ZZ_UPD=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -s 150 -c 1 -o $OUT/${TAG}_upd2 $CMD > $OUT/${TAG}_ncu_upd2.log 2>&1; echo "ncu upd2 $?"
