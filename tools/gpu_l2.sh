#!/bin/bash
# A/B of the L2 eviction priorities in k_update_t (C4), and the DRAM traffic of one fused launch.
OUT=gpurun_out; TAG=${1:-l2}
timeout 300 python -m pytest tests/test_gpu.py -m gpu -x -q -p no:cacheprovider -k "repeat or C2_parity or leading" > $OUT/${TAG}_pytest.log 2>&1; echo "pytest $?"; tail -1 $OUT/${TAG}_pytest.log
for h in 3 5 7 1 3 5 7 1; do
  ZZ_L2HINT=$h timeout 250 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/${TAG}_c4_$h.json 2>&1
  tail -1 $OUT/${TAG}_c4_$h.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hint$h', 'TF %.2f ms %.1f upd %.2f TF share %.3f clk %s' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['share_of_step'], d['clocks']['sm_mhz']))" 2>&1 | tail -1
done
CMD2="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_update_tILi2ELi8ELi1E -s 60 -c 1 -o $OUT/${TAG}_update env ZZ_L2HINT=3 $CMD2 > $OUT/${TAG}_ncu_full.log 2>&1; echo "ncu update exit $?"
