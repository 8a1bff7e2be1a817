#!/bin/bash
# Development: quick timing of the in-tree library against libzz_old.so, and the task timeline
python -c "from paper_2003_04776_b200 import _build; _build.build()"
timeout 300 python -m pytest tests/test_gpu.py -k "${TESTK:-diag_team or C1_parity or power_of_two}" -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/ab_lib.py paper_2003_04776_b200/libzz_old.so paper_2003_04776_b200/libzz.so ${CFGS:-C1:32 C2:128 C3:128 C5:128}
if [ "${TRACE:-1}" = "1" ]; then CFG=C2:128 TEAMS=${TRTEAMS:-0} timeout 300 python tools/trace_team.py; fi
