"""Development: attribute an ncu SASS source page (csv) to CUDA source lines via nvdisasm -g.

  ncu -i X.ncu-rep --page source --csv --print-source sass > sass.csv
  cuobjdump -xelf all build/file.o; nvdisasm -g file.cubin > lines.txt
  python tools/ncu_lines.py sass.csv lines.txt <kernel-substring> <source.cu> [N]
"""
import csv, re, sys
from collections import Counter
sass_csv, lines_txt, kern, srcf = sys.argv[1:5]
N = int(sys.argv[5]) if len(sys.argv) > 5 else 40
L = open(lines_txt).read().splitlines()
start = next(i for i, l in enumerate(L) if l.startswith('//---') and '.text.' in l and kern in l)
end = next((i for i, l in enumerate(L[start + 1:], start + 1) if l.startswith('//---')), len(L))
line = None
off2line = {}
for l in L[start:end]:
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m:
        off2line[int(m.group(1), 16)] = line
rows = list(csv.reader(open(sass_csv)))
h = rows[1]
R = rows[2:]
ai, smp, ie = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
base = int(R[0][ai], 16)
ci, cs = Counter(), Counter()
for r in R:
    ln = off2line.get(int(r[ai], 16) - base)
    ci[ln] += int(r[ie] or 0)
    cs[ln] += int(r[smp] or 0)
ti, ts = sum(ci.values()), sum(cs.values())
import os
srcs = {}
def srcline(ln):
    f, n = ln
    if f not in srcs:
        pth = os.path.join(os.path.dirname(srcf), f)
        srcs[f] = open(pth).read().splitlines() if os.path.exists(pth) else []
    return srcs[f][n - 1].strip()[:90] if n - 1 < len(srcs[f]) else ''
print("line  samples  executed | source")
for ln, n in cs.most_common(N):
    print("%-22s %6.1f%% %6.1f%% | %s" % ("%s:%d" % ln if ln else '-', 100 * n / ts, 100 * ci[ln] / ti, srcline(ln) if ln else ''))
