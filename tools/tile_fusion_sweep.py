"""Development: time to solution over (tile, step-group length, lookahead) on one GPU.

  python tools/tile_fusion_sweep.py C3 [C4 ...] > gpurun_out/<tag>_tf.json
Median of 3 (C4) / 7 (else) timed solves after 2 warm-ups, CUDA events on the solve's
stream; X and the exponents of every variant are compared bit for bit with the first
variant of the same tile (the step-group length and the lookahead never change results)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2003_04776_b200 as zz

VARIANTS = [(128, 4, 1), (128, 6, 1), (96, 4, 1), (96, 6, 1), (64, 4, 1), (64, 6, 1)]
C2_EXTRA = [(128, 4, 2), (64, 4, 2), (64, 6, 2)]
if os.environ.get("TF_VARIANTS"):      # e.g. "32:4:1,32:4:2,64:4:1,64:4:2"
    VARIANTS = [tuple(int(x) for x in v.split(":")) for v in os.environ["TF_VARIANTS"].split(",")]
    C2_EXTRA = []


def main():
    zz.init(0)
    out = []
    for name in sys.argv[1:] or ["C3"]:
        S, T, _ = gen.config(name, seed=0)
        m = S.shape[0]
        Sd = zz.colmajor(torch.from_numpy(S).cuda())
        Td = zz.colmajor(torch.from_numpy(T).cuda())
        del S, T
        X = zz.empty_colmajor(m, m, device="cuda")
        E = torch.empty(m, dtype=torch.int32, device="cuda")
        reps = 3 if m >= 20000 else 7
        ref = {}
        variants = VARIANTS + (C2_EXTRA if m < 4096 else [])
        for mb, fu, la in variants:
            zz.set_tile(mb)
            zz.set_fusion(fu)
            zz.set_lookahead(la)
            for _ in range(2):
                zz.tgevc(Sd, Td, X=X, col_scale_exp=E)
            st = torch.cuda.current_stream()
            ts = []
            for _ in range(reps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(st)
                zz.tgevc(Sd, Td, X=X, col_scale_exp=E)
                b.record(st)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            inf = zz.last_info()
            same = None
            if m < 20000:
                h = (X.cpu().numpy().tobytes(), E.cpu().numpy().tobytes())
                if mb in ref:
                    same = ref[mb] == h
                else:
                    ref[mb] = h
            r = {"config": name, "m": m, "mb": mb, "fusion": fu, "lookahead": la, "median_ms": float(np.median(ts)),
                 "min_ms": float(min(ts)), "launches": inf["total_launches"], "redo": inf.get("lookahead_redo"),
                 "bitwise_vs_first_of_tile": same}
            print(json.dumps(r), file=sys.stderr, flush=True)
            out.append(r)
        del Sd, Td, X
        torch.cuda.empty_cache()
    zz.set_tile(0)
    zz.set_fusion(4)
    zz.set_lookahead(1)
    print(json.dumps({"runs": out}, indent=1))


if __name__ == "__main__":
    main()
