"""Development: solve time per diagonal-solve team size (zz_set_diag_team) and config.

  python tools/time_team.py [lib.so] -- prints config, W, median ms over 5 solves"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch, gen
import paper_2003_04776_b200 as zz
if len(sys.argv) > 1:
    zz._SO = sys.argv[1]
    zz.load(build_if_missing=False)
zz.init(0)
for spec in os.environ.get("CFGS", "C1:32,C2:128,C3:128").split(","):
    name, mb = spec.split(":")
    S, T, _ = gen.config(name, seed=0)
    Sd = zz.colmajor(torch.from_numpy(S).cuda()); Td = zz.colmajor(torch.from_numpy(T).cuda())
    zz.set_tile(int(mb))
    ref = None
    for W in [int(w) for w in os.environ.get("TEAMS", "1,0,3,4,6,12").split(",")]:
        zz.set_diag_team(W)
        X, e = zz.tgevc(Sd, Td); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); zz.tgevc(Sd, Td, X=X, col_scale_exp=e); torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        Xh = X.cpu().numpy()
        same = "" if ref is None else ("bitwise" if np.array_equal(Xh, ref) else "DIFFERENT")
        if ref is None: ref = Xh
        print("%-4s mb=%-4s W=%-3d %9.3f ms %s" % (name, mb, W, 1e3 * float(np.median(ts)), same), flush=True)
    zz.set_diag_team(0)
