"""full-size parity of the GPU path against the oracle, run once.

  python tools/full_parity.py [--config C4] [--chunks 40] [--budget 3000] [--out gpurun_out/x.json]
The GPU solves the whole pencil once (zz_tgevc, the launch configuration bench.py times); the
oracle (oracle/, as it stands, all host cores) then computes the eigenvectors chunk by chunk
(chunk k = the eigenvalue blocks b with b mod chunks == k: every chunk is a stratified sample
over r, so an early stop at the time budget still covers the whole range) and every column is
compared: relative 2-norm difference per eigenvector (a pair as one complex vector), L_c
(Definition 1) relative difference, normalised pairs bitwise (reading R17),
exact zeros below the block, exponents <= 0 and equal within a pair.  The JSON is rewritten
after every chunk.  Test infrastructure (it loads oracle/)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2003_04776_b200 as zz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--chunks", type=int, default=40)
ap.add_argument("--budget", type=float, default=3000.0)   # seconds of oracle time
ap.add_argument("--out", default="")
args = ap.parse_args()

t0 = time.time()
S, T, _ = gen.config(args.config, seed=0)
m = S.shape[0]
tgen = time.time() - t0
zz.init(0)
Sd = zz.colmajor(torch.from_numpy(S).cuda())
Td = zz.colmajor(torch.from_numpy(T).cuda())
X, E = zz.tgevc(Sd, Td)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
zz.tgevc(Sd, Td, X=X, col_scale_exp=E)
e1.record()
torch.cuda.synchronize()
gpu_s = e0.elapsed_time(e1) * 1e-3
info = zz.last_info()
views = zz.last_views()
Eh = E.cpu().numpy()
del Sd, Td
bs, bz = oracle.blocks(S)
nblk = len(bs)
cores = os.cpu_count() or 1
F_all = float(oracle.flops(S))
res = {"config": args.config, "m": m, "blocks": int(nblk), "tile": info["mb"], "gpu_seconds": gpu_s,
       "gpu_tflops": F_all / gpu_s * 1e-12, "oracle_threads": cores, "chunks": args.chunks, "tolerance": 1e-10,
       "gen_seconds": tgen, "chunks_done": 0, "columns_checked": 0, "oracle_seconds": 0.0, "oracle_flops": 0.0,
       "max_rel_2norm": 0.0, "max_logmax_rel": 0.0, "pairs_bitwise": True, "zeros_below": True, "exponents_ok": True,
       "min_exp_gpu": int(Eh.min()), "worst_block_row": -1}
errs = []
for k in range(args.chunks):
    if res["oracle_seconds"] > args.budget:
        break
    ids = np.arange(k, nblk, args.chunks)
    sel = np.zeros(m, np.int32)
    for b in ids:
        sel[bs[b]:bs[b] + bz[b]] = 1
    cols = np.flatnonzero(sel)               # all blocks are computed on the GPU: column == row index
    t1 = time.time()
    r = oracle.tgevc(S, T, select=sel, nthreads=cores)
    dt = time.time() - t1
    assert r["status"] == 0, r["status"]
    res["oracle_seconds"] += dt
    res["oracle_flops"] += float(oracle.flops(S, select=sel))
    Xg = X[:, torch.as_tensor(cols, device=X.device)].cpu().numpy()
    Xo = r["X"]
    c = 0
    for b in ids:
        j, sz = int(bs[b]), int(bz[b])
        if sz == 1:
            a, o = Xg[:, c], Xo[:, c]
        else:
            a, o = Xg[:, c] + 1j * Xg[:, c + 1], Xo[:, c] + 1j * Xo[:, c + 1]
        d = float(np.linalg.norm(a - o) / np.linalg.norm(o))
        errs.append(d)
        if d > res["max_rel_2norm"]:
            res["max_rel_2norm"], res["worst_block_row"] = d, j
        if np.any(Xg[j + sz:, c:c + sz] != 0.0):
            res["zeros_below"] = False
        for q in range(sz):
            g = j + q
            Lg, Lo = views["logmax"][g], r["logmax"][c + q]
            res["max_logmax_rel"] = max(res["max_logmax_rel"], float(abs(Lg - Lo) / max(1.0, abs(Lo))))
            if (views["a"][g], views["b"][g], views["beta"][g]) != tuple(r["pairs"][j]):
                res["pairs_bitwise"] = False
            if Eh[g] > 0 or (sz == 2 and Eh[j] != Eh[j + 1]):
                res["exponents_ok"] = False
        c += sz
    res["chunks_done"] = k + 1
    res["columns_checked"] += int(len(cols))
    res["median_rel_2norm"] = float(np.median(errs))
    res["oracle_gflops"] = res["oracle_flops"] / res["oracle_seconds"] * 1e-9
    res["passed"] = bool(res["max_rel_2norm"] <= 1e-10 and res["max_logmax_rel"] <= 1e-10 and res["pairs_bitwise"]
                         and res["zeros_below"] and res["exponents_ok"])
    if args.out:
        with open(args.out + ".tmp", "w") as f:
            json.dump(res, f, indent=1)
        os.replace(args.out + ".tmp", args.out)
    print("chunk %d/%d: %d columns, oracle %.1f s (total %.0f s), max rel %.3g, L_c %.3g" %
          (k + 1, args.chunks, len(cols), dt, res["oracle_seconds"], res["max_rel_2norm"], res["max_logmax_rel"]),
          file=sys.stderr, flush=True)
res["full"] = res["chunks_done"] == args.chunks
print(json.dumps(res), flush=True)
