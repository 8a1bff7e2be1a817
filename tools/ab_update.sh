#!/bin/bash
# A/B of k_update scheduling variants and the diagonal-solve kernels (development).
OUT=gpurun_out; TAG=${1:-ab}
for cfg in C3 C4; do
for v in "0 0" "0 1" "2 0" "2 1"; do
  set -- $v
  ZZ_UPD_PERSIST=$1 ZZ_UPD_MFAST=$2 timeout 600 python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/${TAG}_${cfg}_p$1_m$2.json 2>&1
  python - $OUT/${TAG}_${cfg}_p$1_m$2.json $cfg $1 $2 <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "persist", sys.argv[3], "mfast", sys.argv[4], "TF %.2f" % d["value"], "ms %.1f" % d["ms_per_step"],
          "upd TF %.2f" % d["roofline"]["achieved"], "upd share %.3f" % d["roofline"]["share_of_step"])
except Exception as e:
    print("fail", sys.argv[1], e, open(sys.argv[1]).read()[-500:])
PY
done
done
