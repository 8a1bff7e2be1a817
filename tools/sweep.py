"""Measurement of SURVEY.md s.8(d)'s per-config protocol on one GPU: time to solution
(median of N after 3 warm-ups, CUDA events on the solve's stream), TFLOP/s = F / t,
the C2 tile sweep and the C3 phase breakdown.  Prints one JSON object.

  python tools/sweep.py > profiles/<round>_sweep.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2003_04776_b200 as zz


def nominal_flops(S):
    m = S.shape[0]
    f, j = 0.0, 0
    while j < m:
        sz = 2 if (j + 1 < m and S[j + 1, j] != 0.0) else 1
        r = j + sz - 1
        f += sz * 2.0 * (r + 1) * r     # 2 r_c (r_c - 1) with 1-based r_c = r + 1
        j += sz
    return f


def run(name, tiles, reps, seed=0):
    S, T, _ = gen.config(name, seed=seed)
    F = nominal_flops(S)
    Sd = zz.colmajor(torch.from_numpy(S).cuda())
    Td = zz.colmajor(torch.from_numpy(T).cuda())
    m = S.shape[0]
    X = zz.empty_colmajor(m, m, device="cuda")
    E = torch.empty(m, dtype=torch.int32, device="cuda")
    out = []
    for mb in tiles:
        zz.set_tile(mb)
        for _ in range(3):
            zz.tgevc(Sd, Td, X=X, col_scale_exp=E)
        ts, ph = [], []
        st = torch.cuda.current_stream()
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            zz.tgevc(Sd, Td, X=X, col_scale_exp=E)
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            ph.append(zz.last_info())
        t = float(np.median(ts))
        inf = ph[len(ph) // 2]
        out.append({"config": name, "m": m, "mb": mb, "tiles": inf["n_tiles"], "median_ms": t,
                    "min_ms": float(min(ts)), "max_ms": float(max(ts)), "reps": reps,
                    "tflops": F / (t * 1e-3) * 1e-12, "F": F,
                    "phase_ms": {k: inf[k] for k in ("ms_setup", "ms_steps", "ms_normalize")},
                    "fused_pairs": inf["fused_pairs"], "launches": inf["total_launches"],
                    "n_scaled_columns": inf["n_scaled"], "min_exp": inf["min_exp"]})
        print(json.dumps(out[-1]), file=sys.stderr)
    return out


if __name__ == "__main__":
    zz.init(0)
    res = {"gpu": torch.cuda.get_device_name(0), "protocol": "median after 3 warm-ups; CUDA events",
           "runs": []}
    res["runs"] += run("C1", [32, 64], 20)
    res["runs"] += run("C2", [32, 64, 96, 128, 160], 20)
    res["runs"] += run("C3", [64, 96, 128, 160], 10)
    res["runs"] += run("C5", [128], 5)
    # C3 with the update kernels timed (phase breakdown incl. the robust-update share)
    zz.set_timing(True)
    r = run("C3", [128], 5)
    zz.set_timing(False)
    inf = zz.last_info()
    r[0]["ms_update"] = inf["ms_update"]
    r[0]["update_share"] = inf["ms_update"] / r[0]["median_ms"]
    r[0]["note"] = "update kernels timed with events (zz_set_timing): phase breakdown"
    res["c3_breakdown"] = r[0]
    print(json.dumps(res, indent=1))
