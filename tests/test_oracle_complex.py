"""Pins of the complex-pencil oracle (oracle/zz_oracle_z.c, ZTGEVC analogue of SURVEY.md
s.8(f) NEXT-4) against things other than itself: LAPACK ZTGEVC as a black box,
the real oracle on real triangular pencils, the m = 1 / m = 2 closed forms, a long-double
unprotected substitution on a stress pencil, and the eigen-residual."""
import numpy as np
import pytest

import gen
import oracle
from tests import lapack_pin

U = 2.0 ** -53


def _resid(S, T, X, alpha, beta):
    R = (S @ X) * beta[None, :] - (T @ X) * alpha[None, :]
    den = (np.abs(beta)[None, :] * np.linalg.norm(S, 1) + np.abs(alpha)[None, :] * np.linalg.norm(T, 1))
    return (np.abs(R).max(axis=0) / (den[0] * np.abs(X).max(axis=0))).max()


@pytest.mark.skipif(not lapack_pin.available(), reason="no LAPACKE in scipy")
@pytest.mark.parametrize("m,seed", [(1, 0), (7, 1), (64, 2), (200, 3)])
def test_ztgevc_matches_lapack(m, seed):
    S, T = gen.complex_pencil(m, seed=seed)
    r = oracle.ztgevc(S, T)
    assert r["status"] == 0
    info, V = lapack_pin.ztgevc(S, T)
    assert info == 0
    # both normalised to max(|Re|+|Im|) = 1 from a real positive tip: the columns are unique
    err = np.abs(r["X"] - V).max(axis=0)
    assert err.max() < 1e3 * m * U, err.max()


@pytest.mark.skipif(not lapack_pin.available(), reason="no LAPACKE in scipy")
def test_ztgevc_select_matches_lapack():
    m = 90
    S, T = gen.complex_pencil(m, seed=5)
    sel = np.zeros(m, np.int32)
    sel[[0, 3, 44, 45, 89]] = 1
    r = oracle.ztgevc(S, T, select=sel)
    info, V = lapack_pin.ztgevc(S, T, select=sel)
    assert info == 0 and r["X"].shape == V.shape == (m, 5)
    assert np.abs(r["X"] - V).max() < 1e3 * m * U


def test_ztgevc_real_pencil_equals_real_oracle():
    """A real upper-triangular pencil is a complex one with zero imaginary parts: the
    eigenvectors must be the real oracle's (real columns, zero imaginary parts)."""
    m = 80
    S, T, _ = gen.generate(m, 0, 1.0 / m, seed=11)
    rr = oracle.tgevc(S, T)
    rz = oracle.ztgevc(S.astype(np.complex128), T.astype(np.complex128))
    assert rr["status"] == 0 and rz["status"] == 0
    assert np.abs(rz["X"].imag).max() == 0.0
    assert np.abs(rz["X"].real - rr["X"]).max() < 64 * U


def test_ztgevc_closed_forms():
    s00, s01, s11 = 0.3 - 0.2j, 0.7 + 0.1j, -0.4 + 0.9j
    t00, t01, t11 = 0.8, -0.25 + 0.5j, 0.6
    S = np.array([[s00, s01], [0, s11]], dtype=np.complex128)
    T = np.array([[t00, t01], [0, t11]], dtype=np.complex128)
    r = oracle.ztgevc(S, T)
    assert r["status"] == 0
    # column 0: e_0; column 1: (s11/t11 eigenvalue) x0 = -(t11 s01 - s11 t01) / (t11 s00 - s11 t00)
    x0 = -(t11 * s01 - s11 * t01) / (t11 * s00 - s11 * t00)
    v = np.array([x0, 1.0])
    v /= np.max(np.abs(v.real) + np.abs(v.imag))
    assert np.allclose(r["X"][:, 0], [1.0, 0.0], rtol=0, atol=0)
    assert np.abs(r["X"][:, 1] - v).max() < 8 * U
    # m = 1: the vector 1; an indefinite eigenvalue (alpha = beta = 0) gives e_j
    r1 = oracle.ztgevc(np.array([[0.5 + 2j]]), np.array([[3.0 + 0j]]))
    assert r1["X"][0, 0] == 1.0
    S0 = np.array([[1.0, 2.0], [0, 0]], dtype=np.complex128)
    T0 = np.array([[1.0, 1.0j], [0, 0]], dtype=np.complex128)
    r0 = oracle.ztgevc(S0, T0)
    assert r0["stats"][2] == 1 and np.array_equal(r0["X"][:, 1], [0.0, 1.0])


def test_ztgevc_status_codes():
    S, T = gen.complex_pencil(6, seed=2)
    T2 = T.copy()
    T2[3, 3] = 1.0 + 1e-3j
    assert oracle.ztgevc(S, T2)["status"] == -107
    S2 = S.copy()
    S2[2, 2] = np.nan
    assert oracle.ztgevc(S2, T)["status"] == -104
    T3 = T.copy()
    T3[1, 1] = -T3[1, 1]                      # negative beta: alpha and beta flip together
    a, be, kd, st = oracle.zeig(S, T3)
    assert st == 0 and (be >= 0).all()


def _longdouble_unprotected(S, T, j):
    """Unprotected substitution in extended precision (exponent range 2^16384: no overflow)."""
    ld = np.clongdouble
    Sl, Tl = S.astype(ld), T.astype(ld)
    al, be = Sl[j, j], Tl[j, j].real
    w = np.zeros(j + 1, dtype=ld)
    w[j] = 1
    for i in range(j - 1, -1, -1):
        rhs = -np.sum((be * Sl[i, i + 1:j + 1] - al * Tl[i, i + 1:j + 1]) * w[i + 1:j + 1])
        w[i] = rhs / (be * Sl[i, i] - al * Tl[i, i])
    return w / np.max(np.abs(w.real) + np.abs(w.imag))


def test_ztgevc_stress_scaling_matches_extended_precision():
    m = 40
    S, T = gen.complex_pencil(m, seed=4, stress=True)
    r = oracle.ztgevc(S, T)
    assert r["status"] == 0 and r["stats"][0] > 0 and np.isfinite(r["X"]).all()
    assert not np.isfinite(oracle.ztgevc(S, T, protect=False)["X"]).all()
    for j in (m - 1, m // 2, 5):
        w = _longdouble_unprotected(S, T, j).astype(np.complex128)
        x = r["X"][: j + 1, j]
        big = np.abs(w) > 1e-250             # entries that survive the rescaling
        assert np.abs(x[big] - w[big]).max() < 1e-10


def test_ztgevc_residual_and_zero_pattern():
    m = 150
    S, T = gen.complex_pencil(m, seed=9)
    r = oracle.ztgevc(S, T)
    a, be, kd, st = oracle.zeig(S, T)
    X = r["X"]
    assert _resid(S, T, X, a, be) < 10 * m * U
    assert np.array_equal(np.tril(X, -1), np.zeros_like(X))
    assert np.allclose((np.abs(X.real) + np.abs(X.imag)).max(axis=0), 1.0, rtol=4 * U, atol=0)
