"""Seeded synthetic Schur pencils (shared input generator; holds none of the method's
arithmetic).  The recipe and the config presets are DESIGN.md section "Inputs"; they stand
in for the paper's starneig-test pencils and follow BASELINE.json configs."""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libzzgen.so")
_lib = None

# BASELINE.json configs[0..4] (readings R16/A10/A11/A14)
CONFIGS = {
    "C1": dict(m=96, n2=24, var_off=1.0 / 96, gap_mode=1, gap=1e-3),
    "C2": dict(m=2000, n2=300, var_off=1.0 / 2000, gap_mode=2, gap=1e-5),
    "C3": dict(m=10000, n2=1500, var_off=1.0 / 10000, gap_mode=2, gap=1e-5),
    "C4": dict(m=40000, n2=6000, var_off=1.0 / 40000, gap_mode=2, gap=1e-5),
    "C5": dict(m=10000, n2=1500, var_off=1.0, gap_mode=0, gap=0.0, stress_frac=0.05,
               stress_tile=128, stress_scale=1e100, cluster=10, cluster_gap=1e-6),
}


def build(force=False):
    src = os.path.join(_HERE, "pencil_gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        f = lib.zzg_generate
        f.restype = ctypes.c_long
        f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_ulonglong, ctypes.c_int,
                      ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                      ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_long,
                      ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        _lib = lib
    return _lib


def generate(m, n2, var_off, seed=0, gap_mode=0, gap=0.0, n_zero=0, n_inf=0, stress_frac=0.0,
             stress_tile=128, stress_scale=1e100, cluster=0, cluster_gap=1e-6, out=None,
             nthreads=0):
    """Return (S, T, lam) with S, T column-major (Fortran-ordered) float64 m x m arrays and
    lam the planted complex eigenvalue per row.  `out=(S_ptr, T_ptr)` writes into caller
    memory (e.g. pinned host tensors, leading dimension m) and returns (None, None, lam)."""
    lib = _load()
    lam_re = np.empty(max(m, 1))
    lam_im = np.empty(max(m, 1))
    if out is None:
        S = np.empty((m, m), order="F")
        T = np.empty((m, m), order="F")
        ps, pt = S.ctypes.data, T.ctypes.data
    else:
        S = T = None
        ps, pt = out
    r = lib.zzg_generate(m, n2, var_off, seed, gap_mode, gap, n_zero, n_inf, stress_frac,
                         stress_tile, stress_scale, cluster, cluster_gap, ps, max(m, 1), pt,
                         max(m, 1), lam_re.ctypes.data, lam_im.ctypes.data, nthreads)
    if r < 0:
        raise RuntimeError("pencil generator failed (separation not reachable or bad args)")
    return S, T, (lam_re + 1j * lam_im)[:m]


def config(name, seed=0, **kw):
    """Generate a BASELINE config pencil ("C1".."C5"), optionally overriding fields."""
    c = dict(CONFIGS[name])
    c.update(kw)
    return generate(seed=seed, **c)


def orthogonal(m, seed=0):
    """Seeded random orthogonal m x m matrix (column-major): the Q factor of a Gaussian
    matrix with the signs of R's diagonal folded in (Haar-distributed).  Stands in for the
    Schur vectors of the QZ step (the back-transformation input, include/zz.h zz_tgevc_back)."""
    rng = np.random.default_rng(1000003 + seed)
    G = rng.standard_normal((m, m))
    Q, R = np.linalg.qr(G)
    d = np.sign(np.diag(R))
    d[d == 0] = 1.0
    return np.asfortranarray(Q * d)


def complex_pencil(m, var_off=None, seed=0, stress=False):
    """Seeded complex Schur pencil (S, T), complex128 column-major m x m, T with a real
    positive diagonal (the ZTGEVC input form).  Built from two real upper-triangular pencils
    of generate() (n2 = 0, off-diagonals N(0, var_off)): S = S1 + i S2, T = T1 + i triu(T2, 1),
    so Re(lambda_j) = S1_jj / T1_jj keeps generate()'s per-eigenvalue separation.
    stress=True multiplies the strictly-upper entries of S by 1e150 in alternate rows so that
    the unprotected substitution overflows (the robust-scaling workload)."""
    if var_off is None:
        var_off = min(1.0, 1.0 / max(m, 1))
    S1, T1, _ = generate(m, 0, var_off, seed=seed)
    S2, T2, _ = generate(m, 0, var_off, seed=seed + 7777)
    S = np.asfortranarray(S1 + 1j * S2)
    T = np.asfortranarray(T1 + 1j * np.triu(T2, 1))
    if stress:
        U = np.triu(np.ones((m, m), dtype=bool), 1)
        U[1::2, :] = False
        S[U] *= 1e150
    return S, T
