python -c "from paper_2003_04776_b200 import _build; _build.build()"
cat > /tmp/gcmp.py <<'PY'
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch, gen, paper_2003_04776_b200 as zz
zz.init(0)
for name, mb in (("C1", 32), ("C2", 128), ("C3", 128)):
    S, T, _ = gen.config(name, seed=0)
    Sd = zz.colmajor(torch.from_numpy(S).cuda()); Td = zz.colmajor(torch.from_numpy(T).cuda())
    m = S.shape[0]
    X = zz.empty_colmajor(m, m); E = torch.empty(m, dtype=torch.int32, device="cuda")
    zz.set_tile(mb)
    for g in (0, 1, 0, 1):
        zz.set_graphs(g)
        for _ in range(3): zz.tgevc(Sd, Td, X=X, col_scale_exp=E)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        reps = 20 if m < 5000 else 5
        e0.record()
        for _ in range(reps): zz.tgevc(Sd, Td, X=X, col_scale_exp=E)
        e1.record(); torch.cuda.synchronize()
        print(name, "graphs", g, "%.3f ms" % (e0.elapsed_time(e1) / reps), flush=True)
PY
timeout 600 python /tmp/gcmp.py
