"""Development: the zero/infinite/indefinite pencil of test_zero_infinite_indefinite_negative,
GPU vs oracle per column (L_c and parity), for the library given as argv[1]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch, gen, oracle
import paper_2003_04776_b200 as zz
from tests import checks
if len(sys.argv) > 1:
    zz._SO = sys.argv[1]; zz.load(build_if_missing=False)
zz.init(0)
S, T, _ = gen.generate(300, 45, 1.0 / 300, seed=11, gap_mode=2, gap=1e-4, n_zero=4, n_inf=5)
d = [j for j in range(1, 299) if S[j, j - 1] == 0 and S[j + 1, j] == 0 and T[j, j] != 0]
T[d[3], d[3]] *= -1
S[d[7], d[7]] = 0.0
T[d[7], d[7]] = 0.0
zz.set_tile(int(os.environ.get("MB", "64")))
zz.set_diag_team(int(os.environ.get("TEAM", "0")))
Sd = zz.colmajor(torch.from_numpy(S).cuda()); Td = zz.colmajor(torch.from_numpy(T).cuda())
X, e = zz.tgevc(Sd, Td); torch.cuda.synchronize()
v = zz.last_views()
X = X.cpu().numpy(); e = e.cpu().numpy()
ref = oracle.tgevc(S, T)
L = v["logmax"]; Lo = ref["logmax"]
dL = np.abs(L - Lo) / np.maximum(1, np.abs(Lo))
lay = checks.column_layout(None, None, S)
raw, ali = checks.parity(X, ref["X"], lay)
bad = np.where(dL > 1e-10)[0]
print("bad L_c columns", bad[:20], "max dL", dL.max(), "max parity", ali.max())
a, b, be, kd, st = oracle.eig_pairs(S, T)
for c in bad[:2]:
    print("col", c, "L", L[c], "Lo", Lo[c], "e", e[c], "eo", ref["e"][c] if "e" in ref else None, "pair", a[c], b[c], be[c])
    nz = np.nonzero(ref["X"][:, c])[0]
    print("   oracle |x| range", np.abs(ref["X"][nz, c]).min(), np.abs(ref["X"][nz, c]).max(), "gpu", np.abs(X[nz, c]).min(), np.abs(X[nz, c]).max())
print("zero/inf rows", [j for j in range(300) if S[j, j] == 0 or T[j, j] == 0])
