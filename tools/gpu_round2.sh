#!/bin/bash
# round evidence: smoke, full GPU tests, default bench, subsets, ncu launch list + full captures,
# per-config sweep, sanitizers
TAG=${1:-r02p}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_gpu.txt 2>&1
python -c "from paper_2003_04776_b200 import _build; _build.build()"
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke exit $?"; tail -2 $OUT/${TAG}_smoke.log
if [ "${TESTS:-1}" = "1" ]; then
timeout 2000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/${TAG}_pytest_gpu.log
fi
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench exit $?"
python -c "import json; d=json.loads(open('$OUT/${TAG}_bench.json').read()); print('C4', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])"
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-roofline --subsets 0.01,0.1 > $OUT/${TAG}_subsets.json 2> $OUT/${TAG}_subsets.err; echo "subsets exit $?"
python -c "import json; d=json.loads(open('$OUT/${TAG}_subsets.json').read()); print(d['subsets'])"
if [ "${SWEEP:-1}" = "1" ]; then
timeout 900 python tools/sweep.py > $OUT/${TAG}_sweep.json 2> $OUT/${TAG}_sweep.err; echo "sweep exit $?"
fi
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-roofline --no-graphs"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/${TAG}_launches.csv $CMD > $OUT/${TAG}_ncu_launches.log 2>&1; echo "ncu launches exit $?"
  CMD2="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-roofline --no-graphs"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k regex:k_update_tILi1E -s 30 -c 1 -o $OUT/${TAG}_update $CMD2 > $OUT/${TAG}_ncu_full.log 2>&1; echo "ncu update exit $?"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k regex:k_diag3 -s 250 -c 1 -o $OUT/${TAG}_diag3_c4 $CMD2 > $OUT/${TAG}_ncu_diag_c4.log 2>&1; echo "ncu diag c4 exit $?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_diag3 -s 20 -c 1 \
      -o $OUT/${TAG}_diag3_c2 python tools/c2_once.py C2 128 > $OUT/${TAG}_ncu_diag_c2.log 2>&1; echo "ncu diag c2 exit $?"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/${TAG}_c2_launches.csv python tools/c2_once.py C2 128 > /dev/null 2>&1; echo "ncu c2 launches exit $?"
fi
if [ "${SAN:-0}" = "1" ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $OUT/${TAG}_san_$tool.log 2>&1; echo "sanitizer $tool exit $?"; tail -3 $OUT/${TAG}_san_$tool.log
  done
fi
if [ "${COMPLEX:-1}" = "1" ]; then
  for M in 2000 4000 10000; do
    timeout 600 python tools/bench_complex.py --m $M > $OUT/${TAG}_complex_$M.json 2> /dev/null
    python -c "import json; d=json.load(open('$OUT/${TAG}_complex_$M.json')); print('complex m=$M', round(d['seconds_per_call']*1e3,2), 'ms', d.get('parity_sample',{}).get('max_abs'))"
  done
  CMDZ="python tools/bench_complex.py --m 10000 --steps 1 --warmup 0 --no-check"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_complex_launches.csv $CMDZ > /dev/null 2>&1; echo "ncu complex launches exit $?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zupdate -s 104 -c 1 -o $OUT/${TAG}_zupdate $CMDZ > /dev/null 2>&1; echo "ncu zupdate exit $?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zdiag -s 120 -c 1 -o $OUT/${TAG}_zdiag $CMDZ > /dev/null 2>&1; echo "ncu zdiag exit $?"
fi
