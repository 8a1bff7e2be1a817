"""Multi-rank run of the collective zz_tgevc / zz_tgevc_host with the in-process transport:
P host threads (ranks) on GPU 0, rank 0 passes S, T, X; X must equal the plain solve bit for
bit.  Prints 'ok P=<P> ...' per case; exits non-zero on a mismatch.
  ZZ_NCCL_LIB=tests/mock_nccl/libmock_nccl.so python tests/mock_nccl/run_ranks.py"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2003_04776_b200 as zz  # noqa: E402


def run(name, P, mb, select_frac=None, **kw):
    S, T, _ = gen.config(name, seed=3, **kw)
    m = S.shape[0]
    sel = None if select_frac is None else (np.random.default_rng(5).random(m) < select_frac).astype(np.int32)
    # the plain solve (a single-rank context on this thread)
    zz.init(0)
    zz.set_tile(mb)
    Sd, Td = zz.colmajor(torch.from_numpy(S).cuda()), zz.colmajor(torch.from_numpy(T).cuda())
    X0, e0 = zz.tgevc(Sd, Td, select=sel)
    torch.cuda.synchronize()
    X0, e0 = X0.cpu().numpy(), e0.cpu().numpy()
    n = X0.shape[1]
    uid = zz.get_unique_id()
    out = {}
    errs = []

    def rank_main(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                zz.init(0, P, r, uid)
                zz.set_tile(mb)
                for host in (False, True):
                    if r == 0:
                        if host:
                            Xh = np.full((m, n), np.nan, order="F")
                            eh = np.zeros(n, np.int32)
                            zz.tgevc_host(S, T, select=sel, X=Xh, col_scale_exp=eh)
                            out["host"] = (Xh, eh)
                        else:
                            X, e = zz.tgevc(Sd, Td, select=sel, n_sel=n)
                            torch.cuda.synchronize()
                            out["dev"] = (X.cpu().numpy(), e.cpu().numpy())
                    else:
                        if host:
                            zz.tgevc_host_collective(m, select=sel)
                        else:
                            zz.tgevc_collective(m, select=sel)
                    torch.cuda.synchronize()
                zz.finalize()
        except Exception as ex:   # noqa: BLE001
            errs.append((r, repr(ex)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs:
        raise RuntimeError(errs)
    for k in ("dev", "host"):
        X, e = out[k]
        if not (np.array_equal(X, X0) and np.array_equal(e, e0)):
            raise SystemExit("MISMATCH %s P=%d %s" % (name, P, k))
    print("ok P=%d %s m=%d n=%d mb=%d" % (P, name, m, n, mb), flush=True)


if __name__ == "__main__":
    assert os.environ.get("ZZ_NCCL_LIB"), "set ZZ_NCCL_LIB to the mock transport"
    run("C1", 2, 32)
    run("C1", 3, 32, select_frac=0.5)
    run("C2", 2, 128)
    run("C2", 3, 64)
    run("C3", 2, 128, m=4096, n2=614)      # lookahead schedule on every rank
    print("all ok")
