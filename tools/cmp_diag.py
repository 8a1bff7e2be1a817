"""Development check: thread-per-eigenvector diagonal solve (default) vs the warp-per-column
kernel (ZZ_DIAG=1, run in a subprocess) vs the oracle; prints parity and timings."""
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(name, seed, mb, out):
    import torch
    import gen
    import paper_2003_04776_b200 as zz
    zz.init(0)
    zz.set_tile(mb)
    S, T, _ = gen.config(name, seed=seed)
    Sd = zz.colmajor(torch.from_numpy(S).cuda())
    Td = zz.colmajor(torch.from_numpy(T).cuda())
    X, e = zz.tgevc(Sd, Td)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        zz.tgevc(Sd, Td, X=X, col_scale_exp=e)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    inf = zz.last_info()
    np.save(out, X.cpu().numpy())
    np.save(out + ".e.npy", e.cpu().numpy())
    return min(ts), inf


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        name, seed, mb, out = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
        t, inf = run(name, seed, mb, out)
        print(json.dumps({"t": t, "info": inf}))
        sys.exit(0)
    import oracle
    import gen
    from tests import checks
    cases = [("C1", 0, 32), ("C1", 3, 64), ("C2", 0, 64), ("C2", 0, 128), ("C2", 1, 96), ("C3", 0, 128),
             ("C5", 0, 128)]
    os.makedirs("gpurun_out", exist_ok=True)
    for name, seed, mb in cases:
        res = {}
        for mode in ("new", "warp"):
            env = dict(os.environ)
            env["ZZ_DIAG"] = "1" if mode == "warp" else os.environ.get("ZZ_DIAG", "3")
            out = "/tmp/cmp_%s_%s.npy" % (name, mode)
            r = subprocess.run([sys.executable, __file__, "child", name, str(seed), str(mb), out], env=env,
                               capture_output=True, text=True)
            if r.returncode != 0:
                print(name, mode, "FAILED", r.stderr[-2000:])
                continue
            res[mode] = (json.loads(r.stdout.strip().splitlines()[-1]), np.load(out), np.load(out + ".e.npy"))
        if len(res) < 2:
            continue
        Xn, Xw = res["new"][1], res["warp"][1]
        line = {"case": "%s s%d mb%d" % (name, seed, mb), "t_new_ms": res["new"][0]["t"] * 1e3,
                "t_warp_ms": res["warp"][0]["t"] * 1e3, "finite": bool(np.isfinite(Xn).all()),
                "n_scaled_new": res["new"][0]["info"]["n_scaled"], "n_scaled_warp": res["warp"][0]["info"]["n_scaled"],
                "bitwise_equal": bool(np.array_equal(Xn, Xw))}
        S, T, _ = gen.config(name, seed=seed)
        lay = checks.column_layout(None, None, S)
        raw, ali = checks.parity(Xn, Xw, lay)
        line["new_vs_warp_max"] = float(ali.max())
        if name != "C5" and S.shape[0] <= 10000:
            ref = oracle.tgevc(S, T)
            raw, ali = checks.parity(Xn, ref["X"], lay)
            line["new_vs_oracle_max"] = float(max(raw.max(), ali.max()))
        print(json.dumps(line), flush=True)
