"""Per-kernel SASS evidence of the in-tree library: counts of the FP64 tensor instruction
(DMMA.8x8x4), TMA tensor loads (UTMALDG), bulk copies (UBLKCP) and tcgen05 MMAs (UTC*MMA: none
-- sm_100a has no FP64 tcgen05 kind).
  python tools/sass_summary.py > profiles/<round>_sass_summary.txt"""
import collections
import os
import re
import subprocess
import sys

so = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                        "paper_2003_04776_b200", "libzz.so")
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
cnt = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        cnt[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    for key, pat in (("DMMA", r"\bDMMA\.8x8x4"), ("UTMALDG", r"\bUTMALDG"), ("UBLKCP", r"\bUBLKCP"), ("UTC*MMA", r"\bUTC\w*MMA")):
        if re.search(pat, line):
            cnt[cur][key] += 1
print("# cuobjdump -sass %s: instruction counts per kernel (kernels with none of them omitted)" % os.path.basename(so))
for k, c in sorted(cnt.items()):
    if sum(c.values()):
        name = re.sub(r"^_ZN?2?z?z?", "", k)
        print("%-100s DMMA %d UTMALDG %d UBLKCP %d UTC*MMA %d" % (name[:100], c["DMMA"], c["UTMALDG"], c["UBLKCP"], c["UTC*MMA"]))
