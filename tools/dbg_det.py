"""Development: determinism bisection (repeat solves in one process) on C3."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch, gen
    import paper_2003_04776_b200 as zz
    zz.init(0); zz.set_tile(128)
    S, T, _ = gen.config(sys.argv[2], seed=0)
    Sd = zz.colmajor(torch.from_numpy(S).cuda()); Td = zz.colmajor(torch.from_numpy(T).cuda())
    outs = []
    for k in range(4):
        X, e = zz.tgevc(Sd, Td); torch.cuda.synchronize()
        outs.append(X.cpu().numpy())
    eq = [np.array_equal(outs[0], o) for o in outs[1:]]
    nbad = [int((np.abs(outs[0] - o).max(axis=0) > 0).sum()) for o in outs[1:]]
    print("repeats equal:", eq, "differing columns:", nbad)
    sys.exit(0)
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
for tag, env in (("nofuse", {"ZZ_FUSE": "1"}), ("pairs", {"ZZ_FUSE": "2"}), ("triples", {"ZZ_FUSE": "3"})):
    cfg = env.get("CFG", cfg)
    r = subprocess.run([sys.executable, __file__, "child", cfg], env=dict(os.environ, **env), capture_output=True, text=True)
    print(tag, "|", r.stdout.strip(), r.stderr[-300:])
