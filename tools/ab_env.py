"""Development: bitwise A/B of two environment settings of the same build on the same inputs.

  python tools/ab_env.py "ZZ_LOOKAHEAD=0" "ZZ_LOOKAHEAD=1" C2:128 C3:128 ...
"""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "child":
    cfg, mb, out = sys.argv[2], int(sys.argv[3]), sys.argv[4]
    import torch, gen
    import paper_2003_04776_b200 as zz
    zz.init(0); zz.set_tile(mb)
    name, _, seed = cfg.partition("@")
    S, T, _ = gen.config(name, seed=int(seed or 0))
    Sd = zz.colmajor(torch.from_numpy(S).cuda()); Td = zz.colmajor(torch.from_numpy(T).cuda())
    X, e = zz.tgevc(Sd, Td); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); zz.tgevc(Sd, Td, X=X, col_scale_exp=e); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    np.save(out, X.cpu().numpy()); np.save(out + ".e.npy", e.cpu().numpy())
    print("%.3f %d" % (1e3 * min(ts), zz.last_info()["n_scaled"]))
    sys.exit(0)
envs = [dict(kv.split("=") for kv in a.split(",") if kv) for a in sys.argv[1:3]]
for spec in sys.argv[3:]:
    cfg, _, mb = spec.partition(":")
    res = []
    for tag, ev in zip("AB", envs):
        out = "/tmp/abe_%s.npy" % tag
        r = subprocess.run([sys.executable, __file__, "child", cfg, mb or "128", out], env=dict(os.environ, **ev),
                           capture_output=True, text=True)
        if r.returncode:
            print(spec, tag, "FAILED", r.stderr[-800:]); break
        t, ns = r.stdout.strip().split()[-2:]
        res.append((float(t), int(ns), np.load(out), np.load(out + ".e.npy")))
    if len(res) == 2:
        (ta, na, Xa, ea), (tb, nb, Xb, eb) = res
        d = np.abs(Xa - Xb)
        print("%-10s A %.3f ms B %.3f ms  scaled %d/%d  bitwise X %s e %s  max|diff| %.3g"
              % (spec, ta, tb, na, nb, np.array_equal(Xa, Xb), np.array_equal(ea, eb), d.max()))
