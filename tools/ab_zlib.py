"""Development: bitwise A/B of builds of libzz.so on the complex path (zz_ztgevc).

  python tools/ab_zlib.py REF.so NEW1.so [NEW2.so ...]
Each library runs in its own process on the same seeded pencils (plain and stress, ragged m,
tiles 64 / 48 / 32, a selection); X and the exponents are compared bit for bit with REF."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

CASES = [(777, 64, 1, False, 0), (777, 64, 2, True, 0), (1500, 64, 4, True, 0), (1000, 48, 3, False, 0),
         (500, 32, 2, True, 0), (2000, 64, 0, False, 1), (1111, 64, 4, True, 1), (65, 64, 1, True, 0), (33, 32, 0, False, 0)]

if len(sys.argv) > 1 and sys.argv[1] == "child":
    lib, out = sys.argv[2], sys.argv[3]
    import torch, gen
    import paper_2003_04776_b200 as zz
    zz._SO = lib
    zz.init(0)
    res = {}
    for n, (m, tile, fusion, stress, sel) in enumerate(CASES):
        S, T = gen.complex_pencil(m, seed=20 + n, stress=stress)
        zz.set_tile(tile)
        if fusion:
            zz.set_fusion(fusion)
        select = None
        if sel:
            select = np.zeros(m, np.int32); select[::3] = 1; select[m - 1] = 1
        Sd = torch.from_numpy(S).cuda().t().contiguous().t(); Td = torch.from_numpy(T).cuda().t().contiguous().t()
        X, E = zz.ztgevc(Sd, Td, select=select)
        torch.cuda.synchronize()
        res["X%d" % n] = X.cpu().numpy(); res["E%d" % n] = E.cpu().numpy()
    np.savez(out, **res)
    sys.exit(0)
ref = None
for lib in sys.argv[1:]:
    out = "/tmp/abz_%s.npz" % os.path.basename(lib)
    r = subprocess.run([sys.executable, __file__, "child", os.path.abspath(lib), out], capture_output=True, text=True)
    if r.returncode:
        print(lib, "FAILED", r.stderr[-800:]); continue
    d = np.load(out)
    if ref is None:
        ref = d; print("ref", lib); continue
    for n, case in enumerate(CASES):
        Xa, Xb, Ea, Eb = ref["X%d" % n], d["X%d" % n], ref["E%d" % n], d["E%d" % n]
        print("%-28s %-34s bitwise X %s E %s  max|diff| %.3g  min E %d" % (os.path.basename(lib), case, np.array_equal(Xa, Xb),
              np.array_equal(Ea, Eb), np.abs(Xa - Xb).max(), Eb.min()))
