#!/bin/bash
timeout 900 python -m pytest tests/test_gpu.py -q -x -p no:cacheprovider -k "lookahead or host_path or fusion_modes_parity" > gpurun_out/la2_pytest.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/la2_pytest.log
for cfg in C3 C4; do for la in 0 1 0 1; do
  ZZ_LOOKAHEAD=$la timeout 250 python bench.py --config $cfg --steps 2 --warmup 2 --no-e2e --no-cpu > gpurun_out/la2_${cfg}_$la.json 2>&1
  tail -1 gpurun_out/la2_${cfg}_$la.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg la$la', 'TF %.2f ms %.2f' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1
done; done
ZZ_LOOKAHEAD=1 timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu > gpurun_out/la2_e2e.json 2>&1; tail -1 gpurun_out/la2_e2e.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 la1 e2e', d['e2e']['value'])"
