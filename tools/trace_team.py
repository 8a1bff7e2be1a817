"""Development: clock64 timeline of one diagonal-solve task (libzz_trace.so, -DZZ_VARIANT_TRACE):
the last k_diag3 launch of a C2 solve, CTA 0, the team's first task."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch, gen
import paper_2003_04776_b200 as zz
zz._SO = os.path.join(os.path.dirname(zz.__file__), "libzz_trace.so")
lib = zz.load(build_if_missing=False)
zz.init(0)
name, mb = os.environ.get("CFG", "C2:128").split(":")
S, T, _ = gen.config(name, seed=0)
Sd = zz.colmajor(torch.from_numpy(S).cuda()); Td = zz.colmajor(torch.from_numpy(T).cuda())
zz.set_tile(int(mb)); zz.set_graphs(False)
for W in [int(w) for w in os.environ.get("TEAMS", "1,12").split(",")]:
    zz.set_diag_team(W)
    for _ in range(2):
        X, e = zz.tgevc(Sd, Td); torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 512)()
    lib.zz_trace_get(buf)
    tr = np.array(buf[:], dtype=np.int64)
    t0 = tr[180]
    rel = lambda v: (v - t0) if v else -1
    print("W=%d  (cycles from kernel start)" % W)
    print("  staged", rel(tr[181]), "bounds", rel(tr[182]))
    print("  init  ", [rel(tr[200 + w]) for w in range(12)])
    print("  chain0", [rel(tr[220 + w]) for w in range(12)])
    for k in range(15, -1, -1):
        print("  blk %2d" % k, [rel(tr[k * 8 + i]) for i in range(7)], "fine", [rel(tr[256 + k * 8 + i]) for i in range(5)])
    print("  epi   ", [rel(tr[140 + w]) for w in range(12)])
    print("  end   ", [rel(tr[160 + w]) for w in range(12)])
