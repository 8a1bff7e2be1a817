"""Development: kernel timeline of one zz_tgevc call from CUPTI activity records (torch.profiler):
per-stream busy time, the gaps on the chain's stream, and how much of the call the bulk update
stream is busy.   python tools/timeline.py C3 [mb]  -> JSON summary on stdout, the raw kernel
list to gpurun_out/timeline_<cfg>.json"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch, gen
import paper_2003_04776_b200 as zz
from torch.profiler import profile, ProfilerActivity

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
mb = int(sys.argv[2]) if len(sys.argv) > 2 else 128
if os.environ.get('ZZ_SO'):
    zz._SO = os.path.abspath(os.environ['ZZ_SO'])
zz.init(0); zz.set_tile(mb)
S, T, _ = gen.config(cfg, seed=0)
Sd = zz.colmajor(torch.from_numpy(S).cuda()); Td = zz.colmajor(torch.from_numpy(T).cuda())
X, E = zz.tgevc(Sd, Td)
for _ in range(3):
    zz.tgevc(Sd, Td, X=X, col_scale_exp=E)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    zz.tgevc(Sd, Td, X=X, col_scale_exp=E)
    torch.cuda.synchronize()
path = "gpurun_out/timeline_%s.trace.json" % cfg
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
os.remove(path)
ks = sorted(({"name": e["name"].split("(")[0][-40:], "stream": e["args"].get("stream"), "ts": e["ts"], "dur": e["dur"],
              "grid": e["args"].get("grid"), "block": e["args"].get("block")} for e in ev), key=lambda k: k["ts"])
t0 = ks[0]["ts"]; t1 = max(k["ts"] + k["dur"] for k in ks)
for k in ks:
    k["ts"] -= t0
json.dump(ks, open("gpurun_out/timeline_%s%s.json" % (cfg, os.environ.get("TAG", "")), "w"))
out = {"config": cfg, "mb": mb, "kernels": len(ks), "span_us": t1 - t0, "streams": {}}
for s in sorted(set(k["stream"] for k in ks)):
    kk = [k for k in ks if k["stream"] == s]
    busy = sum(k["dur"] for k in kk)
    gaps = [kk[i + 1]["ts"] - (kk[i]["ts"] + kk[i]["dur"]) for i in range(len(kk) - 1)]
    byname = {}
    for k in kk:
        n = "k_diag3" if "k_diag3" in k["name"] else ("k_update_t" if "k_update_t" in k["name"] else k["name"])
        byname.setdefault(n, [0, 0.0]); byname[n][0] += 1; byname[n][1] += k["dur"]
    out["streams"][str(s)] = {"kernels": len(kk), "busy_us": busy, "first_us": kk[0]["ts"], "last_end_us": kk[-1]["ts"] + kk[-1]["dur"],
                              "gap_sum_us": float(sum(g for g in gaps if g > 0)), "gap_median_us": float(np.median(gaps)) if gaps else 0.0,
                              "by_kernel": {n: {"launches": v[0], "us": v[1]} for n, v in byname.items()}}
print(json.dumps(out, indent=1))
