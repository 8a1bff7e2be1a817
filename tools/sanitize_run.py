"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck): C1 (tile 32), a
C2-shaped m = 2000 pencil with step groups of 1 and 4 and the lookahead forced on, a stress
pencil (scaling path), the host-staged path, back-transformation, left vectors, the complex
path, and the collective path through a one-rank NCCL communicator with an emulated shard.
  compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2003_04776_b200 as zz  # noqa: E402


def dev(A):
    return zz.colmajor(torch.from_numpy(A).cuda())


zz.init(0)
S, T, _ = gen.config("C1", seed=0)
zz.set_tile(32)
zz.tgevc(dev(S), dev(T))
S2, T2, _ = gen.config("C2", seed=0)
Sd, Td = dev(S2), dev(T2)
zz.set_tile(128)
for fus, la in ((1, 0), (4, 0), (4, 2)):
    zz.set_fusion(fus)
    zz.set_lookahead(la)
    zz.tgevc(Sd, Td)
zz.set_fusion(4)
zz.set_lookahead(1)
c = dict(gen.CONFIGS["C5"])
c.update(m=1000, n2=150, stress_tile=32)
S5, T5, _ = gen.generate(seed=0, **c)
zz.set_tile(64)
zz.tgevc(dev(S5), dev(T5))
zz.tgevc_host(S2, T2)
V = gen.orthogonal(400, seed=1)
S4, T4, _ = gen.config("C2", seed=1, m=400, n2=60)
zz.tgevc_back(dev(S4), dev(T4), dev(V))
zz.tgevc_left(dev(S4), dev(T4))
Sc, Tc = gen.complex_pencil(300, seed=2)
zz.set_tile(64)
zz.ztgevc(torch.from_numpy(Sc).cuda().t().contiguous().t(), torch.from_numpy(Tc).cuda().t().contiguous().t())
zz.init(0, 1, 0, zz.get_unique_id())
zz.set_tile(128)
zz.tgevc(Sd, Td)
zz.set_shard(1, 2)
X = torch.zeros((2000, 2000), dtype=torch.float64, device="cuda").t()
E = torch.zeros(2000, dtype=torch.int32, device="cuda")
zz.tgevc(Sd, Td, X=X, col_scale_exp=E)
zz.set_shard(0, 1)
torch.cuda.synchronize()
zz.init(0)
print("sanitize run ok")
