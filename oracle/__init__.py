"""oracle -- TEST INFRASTRUCTURE ONLY (see oracle/zz_oracle.c header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module.  It wraps the plain C column-by-column robust substitution with ctypes.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libzzoracle.so")
_lib = None


def build(force=False):
    srcs = [os.path.join(_HERE, f) for f in ("zz_oracle.c", "zz_oracle_z.c")]
    if force or not os.path.exists(_SO) or any(os.path.getmtime(_SO) < os.path.getmtime(s) for s in srcs):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", _SO] + srcs + ["-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, ci, cd = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        lib.zzo_protect_update.restype = ci
        lib.zzo_protect_update.argtypes = [cd, cd, cd]
        lib.zzo_protect_division.restype = ci
        lib.zzo_protect_division.argtypes = [cd, cd]
        lib.zzo_blocks.restype = ci
        lib.zzo_blocks.argtypes = [ci, vp, ci, vp, vp]
        lib.zzo_eig_pairs.restype = ci
        lib.zzo_eig_pairs.argtypes = [ci, vp, ci, vp, ci, vp, vp, vp, vp]
        lib.zzo_tgevc_ex.restype = ci
        lib.zzo_tgevc_ex.argtypes = [ci, vp, ci, vp, ci, vp, vp, ci, vp, vp, vp, vp, ci, ci]
        lib.zzo_count_columns.restype = ci
        lib.zzo_count_columns.argtypes = [ci, vp, ci, vp]
        lib.zzo_flops.restype = cd
        lib.zzo_flops.argtypes = [ci, vp, ci, vp]
        lib.zzo_zeig.restype = ci
        lib.zzo_zeig.argtypes = [ci, vp, ci, vp, ci, vp, vp, vp, vp]
        lib.zzo_ztgevc.restype = ci
        lib.zzo_ztgevc.argtypes = [ci, vp, ci, vp, ci, vp, vp, ci, vp, vp, ci, ci]
        _lib = lib
    return _lib


def _f(A):
    A = np.asarray(A, dtype=np.float64)
    if A.ndim != 2 or not A.flags.f_contiguous:
        A = np.asfortranarray(A, dtype=np.float64)
    return A


def _sel(select, m):
    if select is None:
        return None
    s = np.ascontiguousarray(np.asarray(select, dtype=np.int32).reshape(-1))
    assert s.size == m
    return s


def protect_update(y, t, x):
    """exponent e of xi = 2^e = ProtectUpdate(y, t, x)"""
    return _load().zzo_protect_update(y, t, x)


def protect_division(b, t):
    """exponent e of xi = 2^e = ProtectDivision(b, t)"""
    return _load().zzo_protect_division(b, t)


def blocks(S):
    S = _f(S)
    m = S.shape[0]
    bs = np.zeros(max(m, 1), np.int32)
    bz = np.zeros(max(m, 1), np.int32)
    n = _load().zzo_blocks(m, S.ctypes.data, max(m, 1), bs.ctypes.data, bz.ctypes.data)
    if n < 0:
        raise ValueError("status %d" % n)
    return bs[:n].copy(), bz[:n].copy()


def eig_pairs(S, T):
    """per-row normalised (a, b, beta, kind) and the status"""
    S, T = _f(S), _f(T)
    m = S.shape[0]
    a, b, be = (np.zeros(max(m, 1)) for _ in range(3))
    kd = np.zeros(max(m, 1), np.int32)
    st = _load().zzo_eig_pairs(m, S.ctypes.data, max(m, 1), T.ctypes.data, max(m, 1), a.ctypes.data,
                               b.ctypes.data, be.ctypes.data, kd.ctypes.data)
    return a[:m], b[:m], be[:m], kd[:m], st


def count_columns(S, select=None):
    S = _f(S)
    m = S.shape[0]
    sel = _sel(select, m)
    return _load().zzo_count_columns(m, S.ctypes.data, max(m, 1), None if sel is None else sel.ctypes.data)


def flops(S, select=None):
    """nominal F(select) = sum_c 2 r_c (r_c - 1)"""
    S = _f(S)
    m = S.shape[0]
    sel = _sel(select, m)
    return _load().zzo_flops(m, S.ctypes.data, max(m, 1), None if sel is None else sel.ctypes.data)


def tgevc(S, T, select=None, protect=True, nthreads=0):
    """Robust column-by-column eigenvectors.  Returns dict(X, e, logmax, pairs, stats, status);
    X is m x n_sel column-major, e the int32 col_scale_exp, logmax L_c, pairs (m,3)."""
    S, T = _f(S), _f(T)
    m = S.shape[0]
    sel = _sel(select, m)
    lib = _load()
    n = lib.zzo_count_columns(m, S.ctypes.data, max(m, 1), None if sel is None else sel.ctypes.data)
    if n < 0:
        return dict(X=None, e=None, logmax=None, pairs=None, stats=None, status=n)
    X = np.zeros((m, max(n, 1)), order="F")
    e = np.zeros(max(n, 1), np.int32)
    L = np.zeros(max(n, 1))
    pairs = np.zeros((max(m, 1), 3))
    stats = np.zeros(3, np.int32)
    st = lib.zzo_tgevc_ex(m, S.ctypes.data, max(m, 1), T.ctypes.data, max(m, 1),
                          None if sel is None else sel.ctypes.data, X.ctypes.data, max(m, 1),
                          e.ctypes.data, L.ctypes.data, pairs.ctypes.data, stats.ctypes.data,
                          1 if protect else 0, nthreads)
    return dict(X=X[:, :n], e=e[:n], logmax=L[:n], pairs=pairs[:m], stats=stats, status=st)


def tgevc_back(S, T, V, select=None):
    """Back-transformed eigenvectors (xTGEVC HOWMNY='B'; PAPER.md:28-32 read with SURVEY.md A1:
    A (V z) = lambda B (V z) for S = U^T A V, T = U^T B V): W(:, c) = V X(:, c) with X from
    tgevc() above, then LAPACK's normalisation of back-transformed vectors: max |w_i| = 1
    for a real column, max (|Re w_i| + |Im w_i|) = 1 for a complex pair (multiplied by the
    reciprocal of the maximum).  Plain numpy matmul; pinned against LAPACKE_dtgevc with
    HOWMNY='B' (tests/test_oracle_vectors.py)."""
    S, T, V = _f(S), _f(T), _f(V)
    m = S.shape[0]
    r = tgevc(S, T, select=select)
    if r["status"] != 0:
        return dict(W=None, status=r["status"])
    X = r["X"]
    W = np.asfortranarray(V @ X)
    bs, bz = blocks(S)
    sel = _sel(select, m)
    col = 0
    for j, sz in zip(bs, bz):
        if sel is not None and not (sel[j] or (sz == 2 and sel[j + 1])):
            continue
        if sz == 1:
            mx = np.max(np.abs(W[:, col])) if m else 0.0
            if mx > 0:
                W[:, col] *= 1.0 / mx
        else:
            mx = np.max(np.abs(W[:, col]) + np.abs(W[:, col + 1]))
            if mx > 0:
                W[:, col:col + 2] *= 1.0 / mx
        col += sz
    return dict(W=W, X=X, e=r["e"], pairs=r["pairs"], status=0)


def tgevc_left(S, T, select=None):
    """Left eigenvectors y^H S = lambda y^H T (LAPACK xTGEVC SIDE='L').
    Definition used: y^H (beta S - alpha T) = 0  <=>  (beta S^T - conj(alpha) T^T) y = 0; with J
    the reversal, (J S^T J, J T^T J) is a real Schur pencil with the same eigenvalues and
    J conj(y) its right eigenvector for lambda, which tgevc() above computes.  Columns are
    returned in S's block order, a pair as (Re y, Im y) for the eigenvalue with b > 0,
    normalised as the right vectors.  Pinned against LAPACKE_dtgevc(SIDE='L') and the
    left residual (tests/test_oracle_vectors.py)."""
    S, T = _f(S), _f(T)
    m = S.shape[0]
    Sf = np.asfortranarray(S.T[::-1, ::-1])
    Tf = np.asfortranarray(T.T[::-1, ::-1])
    sel = _sel(select, m)
    self_ = None if sel is None else sel[::-1].copy()
    r = tgevc(Sf, Tf, select=self_)
    if r["status"] != 0:
        st = r["status"]
        return dict(Y=None, status=(m - st) if st > 0 else st)
    Xf = r["X"]
    n = Xf.shape[1]
    bs, bz = blocks(Sf)
    kinds = []
    for j, sz in zip(bs, bz):
        if self_ is not None and not (self_[j] or (sz == 2 and self_[j + 1])):
            continue
        kinds += [0] if sz == 1 else [1, 2]
    Y = np.zeros((m, n), order="F")
    e = np.zeros(n, np.int32)
    for c in range(n):
        cc = n - 1 - c
        k = kinds[cc]
        src = cc - 1 if k == 2 else (cc + 1 if k == 1 else cc)
        sg = -1.0 if k == 1 else 1.0
        Y[:, c] = sg * Xf[::-1, src]
        e[c] = r["e"][src]
    return dict(Y=Y, e=e, pairs=r["pairs"][::-1].copy(), status=0)


def _z(A):
    A = np.asarray(A, dtype=np.complex128)
    if A.ndim != 2 or not A.flags.f_contiguous:
        A = np.asfortranarray(A, dtype=np.complex128)
    return A


def zeig(S, T):
    """normalised (alpha, beta) per row of a complex Schur pencil (oracle/zz_oracle_z.c R18):
    returns (alpha complex array, beta, kind, status)"""
    S, T = _z(S), _z(T)
    m = S.shape[0]
    a, b, be = (np.zeros(max(m, 1)) for _ in range(3))
    kd = np.zeros(max(m, 1), np.int32)
    st = _load().zzo_zeig(m, S.ctypes.data, max(m, 1), T.ctypes.data, max(m, 1), a.ctypes.data,
                          b.ctypes.data, be.ctypes.data, kd.ctypes.data)
    return (a + 1j * b)[:m], be[:m], kd[:m], st


def ztgevc(S, T, select=None, protect=True, nthreads=0):
    """Robust column-by-column eigenvectors of a complex Schur pencil (ZTGEVC analogue,
    oracle/zz_oracle_z.c).  Returns dict(X complex m x n_sel, e, stats, status)."""
    S, T = _z(S), _z(T)
    m = S.shape[0]
    sel = _sel(select, m)
    n = m if sel is None else int(np.count_nonzero(sel))
    X = np.zeros((m, max(n, 1)), dtype=np.complex128, order="F")
    e = np.zeros(max(n, 1), np.int32)
    stats = np.zeros(3, np.int32)
    st = _load().zzo_ztgevc(m, S.ctypes.data, max(m, 1), T.ctypes.data, max(m, 1),
                            None if sel is None else sel.ctypes.data, X.ctypes.data, max(m, 1),
                            e.ctypes.data, stats.ctypes.data, 1 if protect else 0, nthreads)
    return dict(X=X[:, :n], e=e[:n], stats=stats, status=st)
