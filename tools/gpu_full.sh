#!/bin/bash
# build, the GPU suite, per-config timing against the previous library
TAG=${1:-r02aa}
OUT=gpurun_out; mkdir -p $OUT
python -c "from paper_2003_04776_b200 import _build; _build.build()"
timeout 2000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/${TAG}_pytest_gpu.log
timeout 900 python tools/ab_lib.py paper_2003_04776_b200/libzz_old.so paper_2003_04776_b200/libzz.so \
    C1:32 C2:128 C3:128 C5:128 C4:128 > $OUT/${TAG}_ab.txt 2>&1; echo "ab exit $?"; cat $OUT/${TAG}_ab.txt
