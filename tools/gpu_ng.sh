#!/bin/bash
# CTA-order grouping of the update kernel (ZZ_NGROUP) A/B on C4, C3; DRAM traffic of one fused launch.
OUT=gpurun_out; TAG=${1:-ng}
timeout 300 python -m pytest tests/test_gpu.py -q -x -p no:cacheprovider -k "repeat or fusion_modes_parity" > $OUT/${TAG}_pytest.log 2>&1; echo "pytest $?"; tail -1 $OUT/${TAG}_pytest.log
for cfg in C4 C3; do
for g in 0 64 32 128 0 64; do
  ZZ_NGROUP=$g timeout 250 python bench.py --config $cfg --steps 2 --warmup 2 --no-e2e --no-cpu > $OUT/${TAG}_${cfg}_$g.json 2>&1
  tail -1 $OUT/${TAG}_${cfg}_$g.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg ng$g', 'TF %.2f ms %.1f upd %.2f TF' % (d['value'], d['ms_per_step'], d['roofline']['achieved']))" 2>&1 | tail -1
done
done
for g in 64 32; do
ZZ_NGROUP=$g timeout 600 ncu --set full --clock-control none --kernel-name-base mangled -k regex:k_update_tILi2ELi8ELi1E -s 40 -c 1 -o $OUT/${TAG}_upd_$g python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > $OUT/${TAG}_ncu_$g.log 2>&1; echo "ncu $g $?"
done
