"""Quick GPU-vs-oracle check (development helper)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import gen, oracle
import paper_2003_04776_b200 as zz
from tests import checks

def run(S, T, mb=0, select=None):
    zz.init(0)
    zz.set_tile(mb)
    Sd = torch.from_numpy(S).cuda(); Td = torch.from_numpy(T).cuda()
    # numpy F-order -> torch: from_numpy keeps strides (column-major)
    X, e = zz.tgevc(Sd, Td, select=select)
    torch.cuda.synchronize()
    return X.cpu().numpy(), e.cpu().numpy(), zz.last_info()

for name, seed, mb in [("C1", 0, 32), ("C1", 1, 32), ("C1", 2, 64), ("C2", 0, 128), ("C2", 0, 64)]:
    S, T, lam = gen.config(name, seed=seed)
    t = time.time(); X, e, info = run(S, T, mb); tg = time.time() - t
    r = oracle.tgevc(S, T)
    lay = checks.column_layout(None, None, S)
    raw, ali = checks.parity(X, r["X"], lay)
    D, B, _ = checks.build_DB(r["pairs"], S)
    res = checks.residual(S, T, X, D, B)
    print(name, seed, mb, "parity raw %.2e ali %.2e" % (raw.max(), ali.max()), "res %.2e" % res, "finite", np.isfinite(X).all(), "e", e.min(), "t %.3f" % tg, info)
    if raw.max() > 1e-8:
        bad = np.argsort(raw)[-3:]
        for b in bad:
            col, j, sz = lay[b]
            print("  bad block", b, "col", col, "row", j, "sz", sz, raw[b])
