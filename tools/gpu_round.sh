#!/bin/bash
# Round evidence (every command under its own timeout): smoke, GPU tests, default bench,
# ncu launch list of one bench step, ncu --set full of k_update and k_diag3 mid-wavefront.
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke exit $?"; tail -1 $OUT/${TAG}_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/${TAG}_pytest_gpu.log
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench exit $?"
cat $OUT/${TAG}_bench.json
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
  timeout 600 $CMD > $OUT/${TAG}_plain.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/${TAG}_launches.csv $CMD > $OUT/${TAG}_ncu_launches.log 2>&1; echo "ncu launches exit $?"
  CMD2="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
  timeout 600 $CMD2 > $OUT/${TAG}_plain2.log 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k regex:k_update_tILi2ELi8ELi1E -s 30 -c 1 \
      -o $OUT/${TAG}_update $CMD2 > $OUT/${TAG}_ncu_full.log 2>&1; echo "ncu update exit $?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_diag -s 150 -c 1 \
      -o $OUT/${TAG}_diag $CMD2 > $OUT/${TAG}_ncu_diag.log 2>&1; echo "ncu diag exit $?"
fi
