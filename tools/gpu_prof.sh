#!/bin/bash
# ncu captures of the two hot kernels (development): k_update mid-wavefront at C4,
# k_diag2 mid-wavefront at C3.  Each command first runs plain and must exit 0.
TAG=${1:-prof}; OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu.py -m gpu -x -q -k "stress or C1 or select or shard" > $OUT/${TAG}_pytest.log 2>&1; echo "pytest $?"; tail -2 $OUT/${TAG}_pytest.log
CMD3="python bench.py --config C3 --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 600 $CMD3 > $OUT/${TAG}_plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_diag2 -s 40 -c 1 -o $OUT/${TAG}_diag2 $CMD3 > $OUT/${TAG}_ncu_diag2.log 2>&1; echo "ncu diag2 $?"
CMD4="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 600 $CMD4 > $OUT/${TAG}_plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -s 150 -c 1 -o $OUT/${TAG}_update $CMD4 > $OUT/${TAG}_ncu_update.log 2>&1; echo "ncu update $?"
