"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list, divided by the
number of API calls in it (the count of a once-per-call marker kernel).
  python tools/launch_split.py gpurun_out/X_launches.csv k_zprep"""
import collections
import csv
import sys

KEYS = ["k_zdiag", "k_zpanel", "k_zprep", "k_zcolmax", "k_znorm", "k_update_t", "k_diag3"]
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
d = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    n = next((k for k in KEYS if k in r[ki]), "library GEMM (cuBLAS/CUTLASS)" if ("gemm" in r[ki].lower() or "cutlass" in r[ki].lower()) else r[ki][:40])
    d[n][0] += 1
    d[n][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
calls = 1
if len(sys.argv) > 2:
    mk = [v[0] for k, v in d.items() if k.startswith(sys.argv[2])]
    calls = max(mk) if mk and max(mk) else 1
tot = sum(v[1] for v in d.values())
print("# %s: per-call device time (ncu, cold-cache, serialised; %d calls in the list)" % (sys.argv[1], calls))
print("%-32s %9s %12s %8s" % ("kernel", "launches", "ms/call", "share"))
for k, v in sorted(d.items(), key=lambda x: -x[1][1]):
    print("%-32s %9d %12.3f %7.2f%%" % (k, v[0] // calls, v[1] / calls, 100 * v[1] / tot))
print("%-32s %9s %12.3f" % ("TOTAL", "", tot / calls))
