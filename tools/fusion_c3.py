"""Development: C3 / C2 time against the step-group length (zz_set_fusion) with the lookahead on."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
import paper_2003_04776_b200 as zz
zz.init(0)
for cfg in sys.argv[1:] or ["C3"]:
    S, T, _ = gen.config(cfg, seed=0)
    Sd = zz.colmajor(torch.from_numpy(S).cuda()); Td = zz.colmajor(torch.from_numpy(T).cuda())
    X, E = zz.tgevc(Sd, Td)
    for mb in (128, 64):
        zz.set_tile(mb)
        for fu in (1, 2, 3, 4, 6):
            zz.set_fusion(fu)
            ts = []
            for it in range(8):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); zz.tgevc(Sd, Td, X=X, col_scale_exp=E); e1.record(); torch.cuda.synchronize()
                if it >= 3: ts.append(e0.elapsed_time(e1))
            print(cfg, "tile", mb, "fusion", fu, "median ms %.3f" % float(np.median(ts)), flush=True)
    zz.set_fusion(0); zz.set_tile(0)
