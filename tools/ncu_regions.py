"""Development: ncu warp-stall samples and executed instructions of one kernel, grouped by
the enclosing function / marked region of a CUDA source file.

  python tools/ncu_regions.py REPORT.ncu-rep OBJECT.o kernel-substring source.cu
"""
import csv, os, re, subprocess, sys, tempfile
from collections import Counter
rep, obj, kern, srcf = sys.argv[1:5]
tmp = tempfile.mkdtemp()
sass = os.path.join(tmp, "sass.csv")
with open(sass, "w") as f:
    subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], stdout=f, check=True)
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
L = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(L) if l.startswith('//---') and '.text.' in l and kern in l)
end = next((i for i, l in enumerate(L[start + 1:], start + 1) if l.startswith('//---')), len(L))
line = None; off2line = {}
for l in L[start:end]:
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m: off2line[int(m.group(1), 16)] = line
rows = list(csv.reader(open(sass)))
h = rows[1]; R = rows[2:]
ai, smp, ie = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
base = int(R[0][ai], 16)
src = open(srcf).read().splitlines()
marks = []
for i, l in enumerate(src, 1):
    if re.match(r'^(template|__device__|__global__|struct)', l) or re.search(r'// ---- ', l):
        marks.append((i, l.strip()[:70]))
def region(ln):
    r = None
    for (i, n) in marks:
        if i <= ln: r = (i, n)
    return r
cs = Counter(); ci = Counter(); ts = ti = 0
for r in R:
    off = int(r[ai], 16) - base; s = float(r[smp] or 0); e = float(r[ie] or 0); ts += s; ti += e
    ln = off2line.get(off)
    key = region(ln[1]) if ln and ln[0] == os.path.basename(srcf) else (0, str(ln[0]) if ln else '?')
    cs[key] += s; ci[key] += e
print("samples %d, instructions executed %d" % (ts, ti))
for k, v in sorted(cs.items(), key=lambda x: -x[1])[:int(sys.argv[5]) if len(sys.argv) > 5 else 25]:
    print("%5.1f%% samples %5.1f%% exec  %s" % (100 * v / ts, 100 * ci[k] / ti, k))
