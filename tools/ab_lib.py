"""Development: bitwise A/B of two builds of libzz.so on the same inputs.

  python tools/ab_lib.py OLD.so NEW.so [config[:mb] ...]
Each library runs in its own process (the binding loads libzz.so by path); X and the
exponents are compared bit for bit, and the solve time of each is printed."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "child":
    lib, cfg, mb, out = sys.argv[2], sys.argv[3], int(sys.argv[4]), sys.argv[5]
    import torch, gen
    import paper_2003_04776_b200 as zz
    zz._SO = lib
    import ctypes
    _CDLL = ctypes.CDLL

    class _Tolerant:               # an older build may lack newer entry points
        def __init__(self, path):
            self._l = _CDLL(path)

        def __getattr__(self, n):
            try:
                return getattr(self._l, n)
            except AttributeError:
                return lambda *a: 0
    ctypes.CDLL = _Tolerant
    zz.load(build_if_missing=False)
    ctypes.CDLL = _CDLL
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
    print("%.3f" % (1e3 * min(ts)))
    sys.exit(0)
old, new = sys.argv[1], sys.argv[2]
for spec in sys.argv[3:] or ["C2:128"]:
    cfg, _, mb = spec.partition(":")
    res = []
    for tag, lib in (("old", old), ("new", new)):
        out = "/tmp/ab_%s.npy" % tag
        r = subprocess.run([sys.executable, __file__, "child", lib, cfg, mb or "128", out], capture_output=True, text=True)
        if r.returncode:
            print(spec, tag, "FAILED", r.stderr[-500:]); break
        res.append((float(r.stdout.strip().splitlines()[-1]), np.load(out), np.load(out + ".e.npy")))
    if len(res) == 2:
        (ta, Xa, ea), (tb, Xb, eb) = res
        d = np.abs(Xa - Xb)
        print("%-10s old %.3f ms new %.3f ms  bitwise X %s e %s  max|diff| %.3g  cols differing %d"
              % (spec, ta, tb, np.array_equal(Xa, Xb), np.array_equal(ea, eb), d.max(), int((d.max(axis=0) > 0).sum())))
