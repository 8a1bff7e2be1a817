#!/bin/bash
# per-config protocol (C1, C2 sweep, C3, C5) + ncu of k_diag3 at C2 (source-level) and C3 launch list
TAG=${1:-r02k}
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2003_04776_b200 import _build; _build.build()"
timeout 900 python tools/sweep.py > $OUT/${TAG}_sweep.json 2> $OUT/${TAG}_sweep.err; echo "sweep exit $?"; cat $OUT/${TAG}_sweep.json | head -c 3000; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_c2_launches.csv python tools/c2_once.py C2 128 > $OUT/${TAG}_c2_ncu.log 2>&1; echo "ncu c2 launches $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_diag3 -s 20 -c 1 -o $OUT/${TAG}_diag3_c2 python tools/c2_once.py C2 128 > $OUT/${TAG}_ncu_diag.log 2>&1; echo "ncu diag $?"
