#!/bin/bash
# lookahead with a bound-based last decision (tree library) against the previous build
# (libzz_old.so): bitwise A/B with timings, the schedule tests, a C4 bench
TAG=${1:-r02at}
OUT=gpurun_out
mkdir -p $OUT
P=paper_2003_04776_b200
for R in 1 2; do python tools/ab_lib.py $P/libzz_old.so $P/libzz.so C3:128 C2:128 C5:128 C1:32 C3:64 C2:64; done 2>&1 | tee $OUT/${TAG}_ab.txt
timeout 1500 python -m pytest tests/test_gpu.py -m gpu -x -q -p no:cacheprovider -k "lookahead or fusion or graph or host or repeat or shard or nccl or multirank or stress or select" > $OUT/${TAG}_pytest_sched.log 2>&1; echo "pytest sched exit $?"; tail -2 $OUT/${TAG}_pytest_sched.log
timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e --no-roofline > $OUT/${TAG}_bench_c4.json 2> /dev/null; python -c "import json; d=json.loads(open('$OUT/${TAG}_bench_c4.json').read()); print('C4', d['ms_per_step'], d['value'])"
