"""Development: a few solves of one config (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_2003_04776_b200 as zz
if os.environ.get("ZZLIB"):          # an alternative build of libzz.so (A/B)
    zz._SO = os.environ["ZZLIB"]
    zz.load(build_if_missing=False)
zz.init(0)
zz.set_graphs(False)   # ncu profiles individual launches
if os.environ.get("TEAM"):
    zz.set_diag_team(int(os.environ["TEAM"]))
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
zz.set_tile(int(sys.argv[2]) if len(sys.argv) > 2 else 128)
S, T, _ = gen.config(name, seed=0)
Sd = zz.colmajor(torch.from_numpy(S).cuda()); Td = zz.colmajor(torch.from_numpy(T).cuda())
for _ in range(2):
    X, e = zz.tgevc(Sd, Td)
torch.cuda.synchronize()
print("ok")
