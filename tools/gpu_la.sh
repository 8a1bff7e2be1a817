#!/bin/bash
# Lookahead A/B: bitwise (no scaling) and time, C1/C2/C3/C5, then C4 bench.
timeout 900 python tools/ab_env.py "ZZ_LOOKAHEAD=0" "ZZ_LOOKAHEAD=1" C1:32 C2:128 C2:64 C3:128 C5:128
timeout 600 python tools/ab_env.py "ZZ_LOOKAHEAD=1,ZZ_LA_PACK=0" "ZZ_LOOKAHEAD=1" C2:128 C3:128
for la in 0 1 0 1; do
  ZZ_LOOKAHEAD=$la timeout 250 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/la_c4_$la.json 2>&1
  tail -1 gpurun_out/la_c4_$la.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 la$la', 'TF %.2f ms %.1f' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1
done
