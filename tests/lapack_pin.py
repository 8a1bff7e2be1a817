"""LAPACK DTGEVC as an independent black-box pin for the oracle (scipy's bundled OpenBLAS
exports LAPACKE_dtgevc; nothing of it is used by the product path or the oracle)."""
import ctypes
import glob
import os

import numpy as np

_f = None


def available():
    return bool(_paths())


def _paths():
    import scipy
    base = os.path.dirname(os.path.dirname(scipy.__file__))
    return glob.glob(os.path.join(base, "scipy.libs", "libscipy_openblas*.so"))


def dtgevc(S, T, select=None):
    """Right eigenvectors (HOWMNY='A' or 'S'); returns (info, VR)."""
    global _f
    if _f is None:
        lib = ctypes.CDLL(_paths()[0])
        _f = lib.scipy_LAPACKE_dtgevc
        _f.restype = ctypes.c_int
    S = np.asfortranarray(S, dtype=np.float64)
    T = np.asfortranarray(T, dtype=np.float64)
    m = S.shape[0]
    VR = np.zeros((m, max(m, 1)), order="F")
    VL = np.zeros((1, 1))
    mo = ctypes.c_int(0)
    if select is None:
        how, sel = b"A", None
    else:
        how = b"S"
        sel = np.ascontiguousarray(np.asarray(select, dtype=np.int32))
    vp = ctypes.c_void_p
    info = _f(102, ctypes.c_char(b"R"), ctypes.c_char(how),
              None if sel is None else sel.ctypes.data_as(vp), m, S.ctypes.data_as(vp), m,
              T.ctypes.data_as(vp), m, VL.ctypes.data_as(vp), 1, VR.ctypes.data_as(vp), m, m,
              ctypes.byref(mo))
    return info, VR[:, :mo.value]


def dtgevc_back(S, T, V):
    """Back-transformed right eigenvectors (HOWMNY='B', VR = V on entry); returns (info, VR)."""
    global _f
    if _f is None:
        lib = ctypes.CDLL(_paths()[0])
        _f = lib.scipy_LAPACKE_dtgevc
        _f.restype = ctypes.c_int
    S = np.asfortranarray(S, dtype=np.float64)
    T = np.asfortranarray(T, dtype=np.float64)
    m = S.shape[0]
    VR = np.array(V, dtype=np.float64, order="F", copy=True)
    VL = np.zeros((1, 1))
    mo = ctypes.c_int(0)
    vp = ctypes.c_void_p
    info = _f(102, ctypes.c_char(b"R"), ctypes.c_char(b"B"), None, m, S.ctypes.data_as(vp), m,
              T.ctypes.data_as(vp), m, VL.ctypes.data_as(vp), 1, VR.ctypes.data_as(vp), m, m,
              ctypes.byref(mo))
    return info, VR[:, :mo.value]


def dtgevc_left(S, T, select=None):
    """Left eigenvectors (SIDE='L', HOWMNY='A' or 'S'); returns (info, VL)."""
    global _f
    if _f is None:
        lib = ctypes.CDLL(_paths()[0])
        _f = lib.scipy_LAPACKE_dtgevc
        _f.restype = ctypes.c_int
    S = np.asfortranarray(S, dtype=np.float64)
    T = np.asfortranarray(T, dtype=np.float64)
    m = S.shape[0]
    VL = np.zeros((m, max(m, 1)), order="F")
    VR = np.zeros((1, 1))
    mo = ctypes.c_int(0)
    if select is None:
        how, sel = b"A", None
    else:
        how = b"S"
        sel = np.ascontiguousarray(np.asarray(select, dtype=np.int32))
    vp = ctypes.c_void_p
    info = _f(102, ctypes.c_char(b"L"), ctypes.c_char(how),
              None if sel is None else sel.ctypes.data_as(vp), m, S.ctypes.data_as(vp), m,
              T.ctypes.data_as(vp), m, VL.ctypes.data_as(vp), m, VR.ctypes.data_as(vp), 1, m,
              ctypes.byref(mo))
    return info, VL[:, :mo.value]


def ztgevc(S, T, select=None):
    """LAPACK ZTGEVC right eigenvectors (HOWMNY='A' or 'S'); returns (info, VR complex)."""
    lib = ctypes.CDLL(_paths()[0])
    f = lib.scipy_LAPACKE_ztgevc
    f.restype = ctypes.c_int
    S = np.asfortranarray(S, dtype=np.complex128)
    T = np.asfortranarray(T, dtype=np.complex128)
    m = S.shape[0]
    VR = np.zeros((m, max(m, 1)), dtype=np.complex128, order="F")
    VL = np.zeros((1, 1), dtype=np.complex128)
    mo = ctypes.c_int(0)
    if select is None:
        how, sel = b"A", None
    else:
        how = b"S"
        sel = np.ascontiguousarray(np.asarray(select, dtype=np.int32))
    vp = ctypes.c_void_p
    info = f(102, ctypes.c_char(b"R"), ctypes.c_char(how),
             None if sel is None else sel.ctypes.data_as(vp), m, S.ctypes.data_as(vp), m,
             T.ctypes.data_as(vp), m, VL.ctypes.data_as(vp), 1, VR.ctypes.data_as(vp), m, m,
             ctypes.byref(mo))
    return info, VR[:, :mo.value]
