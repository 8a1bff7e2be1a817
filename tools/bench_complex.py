"""Timing of zz_ztgevc (complex pencils) on one GPU.

python tools/bench_complex.py --m 10000 --steps 3 --warmup 2
Prints one JSON line: seconds per call (CUDA events on the launching stream, inputs
resident in HBM, larger than L2 at m >= 4000), nominal flops F_z = sum_j 8 j (j + 1)
(every (i, k) pair i < k <= j of column j costs two complex multiply-adds = 16 flop), the
FP64 fraction against the DMMA peak, and a sampled parity check against the oracle."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2003_04776_b200 as zz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=10000)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--no-check", action="store_true")
ap.add_argument("--lookahead", type=int, default=1)
ap.add_argument("--fusion", type=int, default=0)   # 0: the library default (by the number of tile rows)
ap.add_argument("--lib", default="")   # development: another build of libzz.so (A/B)
ap.add_argument("--full-check", action="store_true",
                help="compare EVERY column with the oracle (stratified chunks of the columns; m = 10000: about a minute of host time)")
args = ap.parse_args()

m = args.m
t0 = time.time()
S, T = gen.complex_pencil(m, seed=args.seed)
tgen = time.time() - t0
if args.lib:
    zz._SO = os.path.abspath(args.lib)
zz.init(0)
zz.set_tile(args.tile)
zz.set_lookahead(args.lookahead)
if args.fusion:
    zz.set_fusion(args.fusion)
Sd = torch.from_numpy(S).cuda().t().contiguous().t()
Td = torch.from_numpy(T).cuda().t().contiguous().t()
st = torch.cuda.current_stream()
X, E = zz.ztgevc(Sd, Td)
for _ in range(args.warmup):
    zz.ztgevc(Sd, Td, X=X, col_scale_exp=E)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(args.steps):
    zz.ztgevc(Sd, Td, X=X, col_scale_exp=E)
e1.record(st)
torch.cuda.synchronize()
sec = e0.elapsed_time(e1) / 1e3 / args.steps
j = np.arange(m, dtype=np.float64)
F = float(np.sum(8.0 * j * (j + 1.0)))
info = zz.last_info()
out = {"metric": "seconds & FP64 TFLOP/s, all eigenvectors of a complex Schur pencil (zz_ztgevc)",
       "m": m, "tile": info["mb"], "steps": args.steps, "warmup": args.warmup,
       "seconds_per_call": sec, "flops_nominal": F, "value": F / sec * 1e-12, "unit": "TFLOP/s",
       "update_product": "gauss3m (k_zupdate, three DMMA contractions)", "lookahead": args.lookahead, "fusion": args.fusion,
       # the Gauss 3M update executes 3/4 of F_z's real flops: the first ratio is an effective
       # (time-to-solution) figure, the second the executed flops' share of the DMMA peak
       "effective_fraction_nominal_flops": F / sec * 1e-12 / 37.0,
       "executed_fraction_3m_flops": 0.75 * F / sec * 1e-12 / 37.0,
       "peak_source": "DMMA FP64 37.0 TFLOP/s measured (profiles/r01_fp64_peak.json)",
       "launches_per_call": info["total_launches"], "update_launches": info["update_launches"],
       "data": "synthetic: gen.complex_pencil (two real generate() pencils, off-diagonals N(0,1/m))",
       "gen_seconds": tgen}
if not args.no_check:
    import oracle
    cols = sorted(set([0, m // 3, m // 2, m - 2, m - 1]))
    sel = np.zeros(m, np.int32)
    sel[cols] = 1
    ref = oracle.ztgevc(S, T, select=sel)
    Xh = X[:, cols].cpu().numpy()
    out["parity_sample"] = {"columns": cols, "max_abs": float(np.abs(Xh - ref["X"]).max()), "tolerance": 1e-10}
    # the oracle as it stands, on the host cores, on a stratified sample of 96 columns
    samp = np.unique(np.linspace(0, m - 1, 96).astype(np.int64))
    sel2 = np.zeros(m, np.int32)
    sel2[samp] = 1
    Fs = float(np.sum(8.0 * samp.astype(np.float64) * (samp + 1.0)))
    t0 = time.time()
    oracle.ztgevc(S, T, select=sel2)
    tc = time.time() - t0
    out["cpu_baseline"] = {"value": Fs / tc * 1e-12, "unit": "TFLOP/s", "cores": os.cpu_count(),
                           "kind": "oracle", "seconds": tc,
                           "sample": "%d columns evenly spaced over j of the same pencil, F_sample = %.3g flop"
                                     % (len(samp), Fs)}
if args.full_check:
    import oracle
    nch = max(1, m // 1000)
    Eh = E.cpu().numpy()
    worst, tor, zeros_ok = 0.0, 0.0, True
    for k in range(nch):
        cols = np.arange(k, m, nch)
        selk = np.zeros(m, np.int32)
        selk[cols] = 1
        t0 = time.time()
        ref = oracle.ztgevc(S, T, select=selk)
        tor += time.time() - t0
        assert ref["status"] == 0
        Xg = X[:, torch.as_tensor(cols, device=X.device)].cpu().numpy()
        worst = max(worst, float(np.abs(Xg - ref["X"]).max()))
        for q, j in enumerate(cols):
            if np.any(Xg[j + 1:, q] != 0):
                zeros_ok = False
    out["parity_full"] = {"columns": m, "chunks": nch, "max_abs": worst, "tolerance": 1e-10, "zeros_below": zeros_ok,
                          "exponents_nonpositive": bool((Eh <= 0).all()), "oracle_seconds": tor, "oracle_threads": os.cpu_count(),
                          "oracle_tflops_nominal": F / tor * 1e-12, "passed": bool(worst <= 1e-10 and zeros_ok and (Eh <= 0).all())}
print(json.dumps(out), flush=True)
