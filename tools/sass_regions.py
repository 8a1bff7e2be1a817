"""Development: SASS instruction count of one kernel per source region (function or '// ---- '
marker) from nvdisasm line info.   python tools/sass_regions.py OBJ.o kernel-substring source.cu [N]"""
import os, re, subprocess, sys, tempfile
from collections import Counter
obj, kern, srcf = sys.argv[1:4]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 20
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
L = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout.splitlines()
src = open(srcf).read().splitlines()
marks = [(i, l.strip()[:70]) for i, l in enumerate(src, 1)
         if re.match(r'^(template|__device__|__global__|struct)', l) or re.search(r'// ---- ', l)]
def region(ln):
    r = None
    for (i, n) in marks:
        if i <= ln: r = (i, n)
    return r
start = next(i for i, l in enumerate(L) if l.startswith('//---') and '.text.' in l and kern in l)
end = next((i for i, l in enumerate(L[start + 1:], start + 1) if l.startswith('//---')), len(L))
c = Counter(); line = None; n = 0
for l in L[start:end]:
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1).split('/')[-1], int(m.group(2))); continue
    if re.search(r'/\*([0-9a-f]{4,})\*/\s', l) and not l.strip().startswith('/*0'):
        pass
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/\s+\S', l):
        n += 1
        key = region(line[1]) if line and line[0] == os.path.basename(srcf) else (0, line[0] if line else '?')
        c[key] += 1
print(kern, "SASS instructions", n)
for k, v in c.most_common(N): print("  %6d  %s" % (v, k))
