"""Development: time the solve with the diagonal-solve kernel chosen by ZZ_DIAG (1 = warp per
eigenvector k_diag, 3 = k_diag3) per config; one process per setting."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch, gen
    import paper_2003_04776_b200 as zz
    zz.init(0)
    out = []
    for spec in sys.argv[2:]:
        name, _, mb = spec.partition(":")
        zz.set_tile(int(mb or 128))
        S, T, _ = gen.config(name, seed=0)
        Sd = zz.colmajor(torch.from_numpy(S).cuda()); Td = zz.colmajor(torch.from_numpy(T).cuda())
        X, e = zz.tgevc(Sd, Td); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); zz.tgevc(Sd, Td, X=X, col_scale_exp=e); torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out.append("%s %.3f ms" % (spec, 1e3 * sorted(ts)[2]))
    print(" | ".join(out))
    sys.exit(0)
for kind in ("3", "1"):
    r = subprocess.run([sys.executable, __file__, "child"] + sys.argv[1:], env=dict(os.environ, ZZ_DIAG=kind),
                       capture_output=True, text=True)
    print("ZZ_DIAG=%s:" % kind, r.stdout.strip(), r.stderr[-300:] if r.returncode else "")
