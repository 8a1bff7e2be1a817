"""Pins of the oracle's eigenvectors (oracle/zz_oracle.c) against things other than itself:
closed forms (m = 1, 2), long-double brute-force null vectors (m <= 8),
LAPACK DTGEVC as a black box, a long-double unprotected substitution on stress pencils,
and the invariants of DESIGN.md (residual, zeros, exponents, equivariance, independence)."""
import numpy as np
import pytest

import gen
import oracle
from tests import checks
from tests import lapack_pin

U = 2.0 ** -53


def _run(S, T, select=None, protect=True):
    r = oracle.tgevc(S, T, select=select, protect=protect)
    assert r["status"] == 0
    return r


def _norm(z):
    return z / np.max(np.abs(z.real) + np.abs(z.imag))


def test_m1():
    r = _run(np.array([[2.0]], order="F"), np.array([[1.0]], order="F"))
    assert r["X"].tolist() == [[1.0]] and r["e"].tolist() == [0]


def test_m0():
    r = oracle.tgevc(np.zeros((0, 0), order="F"), np.zeros((0, 0), order="F"))
    assert r["status"] == 0 and r["X"].shape == (0, 0)


def test_triangular_2x2_closed_form():
    # eigenvector of lambda2 = s22/t22: (-(t22 s12 - s22 t12) / (t22 s11 - s22 t11), 1)
    s11, s12, s22, t11, t12, t22 = 0.7, -1.3, -0.4, 1.1, 0.25, 0.9
    S = np.array([[s11, s12], [0, s22]], order="F")
    T = np.array([[t11, t12], [0, t22]], order="F")
    X = _run(S, T)["X"]
    v = np.array([-(t22 * s12 - s22 * t12) / (t22 * s11 - s22 * t11), 1.0])
    v /= np.max(np.abs(v))
    assert np.allclose(X[:, 1], v, rtol=1e-15, atol=1e-16)
    assert np.allclose(X[:, 0], [1.0, 0.0])


def test_spec_diag_identity():
    # S = diag(1,2,3), T = I -> V = I
    X = _run(np.diag([1.0, 2.0, 3.0]).copy(order="F"), np.eye(3, order="F"))["X"]
    assert np.array_equal(X, np.eye(3))


def test_spec_tile_example():
    # S=[[1,1],[0,2]], T=I, eigenvalue 2 -> (1,1)
    X = _run(np.array([[1.0, 1.0], [0, 2.0]], order="F"), np.eye(2, order="F"))["X"]
    assert np.allclose(X[:, 1], [1.0, 1.0], rtol=0, atol=1e-15)


def test_spec_rotation_tip_phase_aligned():
    # S=[[0,1],[-1,0]], T=I -> z proportional to (1, i)
    X = _run(np.array([[0.0, 1.0], [-1.0, 0.0]], order="F"), np.eye(2, order="F"))["X"]
    z = X[:, 0] + 1j * X[:, 1]
    ref = np.array([1.0, 1j])
    c = np.vdot(ref, z) / abs(np.vdot(ref, z))
    assert np.allclose(z, c * ref / 1.0, atol=1e-15)
    assert np.max(np.abs(X[:, 0]) + np.abs(X[:, 1])) == 1.0


def _random_small(m, seed, n2=None, zeros=0, infs=0):
    rng = np.random.default_rng(seed)
    n2 = rng.integers(0, m // 2 + 1) if n2 is None else n2
    S, T, _ = gen.generate(m, int(n2), 1.0 / m, seed=seed, n_zero=zeros, n_inf=infs)
    return S, T


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("seed", range(6))
def test_brute_force_long_double(m, seed):
    S, T = _random_small(m, 1000 * m + seed, zeros=(seed == 4), infs=(seed == 5))
    r = _run(S, T)
    lay = checks.column_layout(None, None, S)
    zs = checks.to_complex(r["X"], lay)
    for z, (col, j, sz) in zip(zs, lay):
        a, b, be = r["pairs"][j]
        if a == 0 and b == 0 and be == 0:
            continue
        ref = checks.brute_null_vector(S, T, a, b, be)
        # same direction up to a complex scalar (the brute force fixes its own phase)
        c = np.vdot(ref, z) / np.vdot(ref, ref)
        err = np.linalg.norm(z - c * ref) / np.linalg.norm(z)
        assert err < 1e-12, (m, seed, j, err)


def _lapack_or_skip():
    if not lapack_pin.available():
        pytest.skip("scipy OpenBLAS LAPACKE not available")


@pytest.mark.parametrize("seed", range(10))
def test_lapack_dtgevc_C1(seed):
    _lapack_or_skip()
    S, T, _ = gen.config("C1", seed=seed)
    r = _run(S, T)
    info, VR = lapack_pin.dtgevc(S, T)
    assert info == 0
    lay = checks.column_layout(None, None, S)
    raw, ali = checks.parity(r["X"], VR, lay)
    assert ali.max() < 1e-11 and raw.max() < 1e-11


@pytest.mark.parametrize("m,n2,zeros,infs", [(500, 75, 5, 5), (1000, 150, 10, 10)])
def test_lapack_dtgevc_larger_with_zero_inf(m, n2, zeros, infs):
    _lapack_or_skip()
    S, T, _ = gen.generate(m, n2, 1.0 / m, seed=7, gap_mode=2, gap=1e-4, n_zero=zeros, n_inf=infs)
    r = _run(S, T)
    info, VR = lapack_pin.dtgevc(S, T)
    assert info == 0
    lay = checks.column_layout(None, None, S)
    raw, ali = checks.parity(r["X"], VR, lay)
    assert ali.max() < 1e-10, ali.max()


def test_lapack_selected_subset():
    _lapack_or_skip()
    S, T, _ = gen.config("C1", seed=3)
    m = S.shape[0]
    sel = np.zeros(m, np.int32)
    sel[[0, 5, 17, 40, 41, 77, 95]] = 1
    r = _run(S, T, select=sel)
    info, VR = lapack_pin.dtgevc(S, T, select=sel)
    assert info == 0 and VR.shape == r["X"].shape
    lay = checks.column_layout(None, None, S, sel)
    raw, ali = checks.parity(r["X"], VR, lay)
    assert raw.max() < 1e-11


def test_lapack_info_real_2x2_and_indefinite():
    _lapack_or_skip()
    # real eigenvalues in a 2x2 block: oracle and DTGEVC both report the 1-based row
    S = np.array([[0.5, 0.1, 0.2], [0.0, 1.0, 0.3], [0.0, 1.0, 1.0]], order="F")
    T = np.eye(3, order="F")
    assert oracle.tgevc(S, T)["status"] == 2
    info, _ = lapack_pin.dtgevc(S, T)
    assert info == 2
    # indefinite 1x1 (S_jj = T_jj = 0) -> unit vector e_j (DTGEVC behaviour)
    S = np.array([[0.5, 0.1, 0.2], [0.0, 0.0, 0.3], [0.0, 0.0, 1.0]], order="F")
    T = np.array([[1.0, 0.2, 0.1], [0.0, 0.0, 0.4], [0.0, 0.0, 2.0]], order="F")
    r = _run(S, T)
    info, VR = lapack_pin.dtgevc(S, T)
    assert info == 0
    assert np.array_equal(r["X"][:, 1], [0.0, 1.0, 0.0])
    assert np.allclose(VR[:, 1], [0.0, 1.0, 0.0])


@pytest.mark.parametrize("name,seed", [("C1", 0), ("C1", 1), ("C2", 0)])
def test_invariants(name, seed):
    S, T, _ = gen.config(name, seed=seed)
    m = S.shape[0]
    r = _run(S, T)
    X, e = r["X"], r["e"]
    assert np.isfinite(X).all()
    assert (e <= 0).all()
    D, B, lay = checks.build_DB(r["pairs"], S)
    for col, j, sz in lay:
        rlast = j + sz - 1
        assert np.all(X[rlast + 1:, col:col + sz] == 0.0)
        if sz == 2:
            assert e[col] == e[col + 1]
            assert abs(np.max(np.abs(X[:, col]) + np.abs(X[:, col + 1])) - 1.0) <= 2 * U
        else:
            assert abs(np.max(np.abs(X[:, col])) - 1.0) <= 2 * U
    res = checks.residual(S, T, X, D, B)
    assert res <= 10 * m * U, res
    assert checks.comp_backward_error(S, T, X, r["pairs"], lay, m) <= 10 * m * U


def test_power_of_two_equivariance_bitwise():
    S, T, _ = gen.config("C1", seed=2)
    r0 = _run(S, T)
    for k in (-300, -7, 5, 200):
        r1 = _run(np.ldexp(S, k), np.ldexp(T, k))
        assert np.array_equal(r0["X"], r1["X"])


def test_column_independence_bitwise():
    S, T, _ = gen.config("C1", seed=4)
    m = S.shape[0]
    r0 = _run(S, T)
    lay = checks.column_layout(None, None, S)
    for col, j, sz in lay[::7]:
        sel = np.zeros(m, np.int32)
        sel[j] = 1
        r1 = _run(S, T, select=sel)
        assert np.array_equal(r1["X"], r0["X"][:, col:col + sz])


def test_thread_count_independence():
    S, T, _ = gen.config("C2", seed=1)
    r1 = oracle.tgevc(S, T, nthreads=1)
    r4 = oracle.tgevc(S, T, nthreads=4)
    assert np.array_equal(r1["X"], r4["X"]) and np.array_equal(r1["e"], r4["e"])


def test_prescale_path_large_entries():
    # entries near Omega/4: the row-sum norm exceeds Omega/8, the oracle
    # pre-scales by a power of two; eigenvectors equal those of the unscaled pencil.
    S, T, _ = gen.config("C1", seed=5)
    big = 2.0 ** 1021
    r0 = _run(S, T)
    r1 = _run(S * big, T * big)
    assert np.array_equal(r0["X"], r1["X"])


# ------------------------- overflow protection (stress) -------------------------

def _ld_substitution(S, T, a, b, beta, j, sz):
    """unprotected substitution in long double (15-bit exponent), tip rule of DESIGN R10"""
    r = j + sz - 1
    Sl = np.asarray(S, dtype=np.longdouble)
    Tl = np.asarray(T, dtype=np.longdouble)
    al = np.clongdouble(complex(a, b))
    be = np.longdouble(beta)
    z = np.zeros(r + 1, dtype=np.clongdouble)
    if sz == 1:
        z[r] = 1
    else:
        p = be * Sl[r, r - 1]
        q = be * Sl[r, r] - al * Tl[r, r]
        if abs(p) >= abs(q.real) + abs(q.imag):
            z[r] = 1
            z[r - 1] = -q / p
        else:
            z[r - 1] = 1
            z[r] = -p / q
    top = r - sz + 1
    z[:top] -= (be * Sl[:top, top:r + 1] - al * Tl[:top, top:r + 1]) @ z[top:r + 1]
    i = top - 1
    while i >= 0:
        two = i >= 1 and S[i, i - 1] != 0.0
        if not two:
            d = be * Sl[i, i] - al * Tl[i, i]
            z[i] = z[i] / d
            z[:i] -= (be * Sl[:i, i] - al * Tl[:i, i]) * z[i]
            i -= 1
        else:
            k = i - 1
            C = be * Sl[k:i + 1, k:i + 1] - al * Tl[k:i + 1, k:i + 1]
            det = C[0, 0] * C[1, 1] - C[0, 1] * C[1, 0]
            y0, y1 = z[k], z[i]
            z[k] = (C[1, 1] * y0 - C[0, 1] * y1) / det
            z[i] = (C[0, 0] * y1 - C[1, 0] * y0) / det
            z[:k] -= (be * Sl[:k, k:i + 1] - al * Tl[:k, k:i + 1]) @ z[k:i + 1]
            i -= 2
    return z


def _stress(m, seed, tile=32):
    c = dict(gen.CONFIGS["C5"])
    c.update(m=m, n2=int(0.15 * m), stress_tile=tile)
    S, T, _ = gen.generate(seed=seed, **c)
    return S, T


def test_stress_negative_control_and_robust():
    S, T = _stress(1000, 0)
    rn = oracle.tgevc(S, T, protect=False)
    bad = (~np.isfinite(rn["X"]).all(axis=0)).sum()
    assert bad > 0  # naive substitution overflows
    r = _run(S, T)
    assert np.isfinite(r["X"]).all()
    assert (r["e"] <= 0).all() and (r["e"] < 0).sum() >= bad
    lay = checks.column_layout(None, None, S)
    assert checks.comp_backward_error(S, T, r["X"], r["pairs"], lay, S.shape[0]) <= 10 * 1000 * U


def test_stress_exponents_vs_long_double():
    S, T = _stress(400, 1, tile=16)
    r = _run(S, T)
    assert (r["e"] < 0).sum() > 20
    lay = checks.column_layout(None, None, S)
    zs = checks.to_complex(r["X"], lay)
    checked = 0
    for z, (col, j, sz) in zip(zs, lay):
        if (r["e"][col] == 0 and checked > 10) or checked > 60:
            continue
        a, b, be = r["pairs"][j]
        zl = _ld_substitution(S, T, a, b, be, j, sz)
        mx = np.max(np.abs(zl.real) + np.abs(zl.imag)) if sz == 2 else np.max(np.abs(zl.real))
        L = float(np.log2(mx))
        assert abs(L - r["logmax"][col]) <= 1e-12 * max(1.0, abs(L)), (j, L, r["logmax"][col])
        zn = (zl / mx).astype(complex)
        ref = np.zeros(S.shape[0], complex)
        ref[:zn.size] = zn
        assert np.linalg.norm(z - ref) / np.linalg.norm(ref) < 1e-9
        checked += 1
    assert checked > 30


def test_stress_c5_recipe_small_scale():
    c = dict(gen.CONFIGS["C5"])
    c.update(m=2000, n2=300)
    S, T, _ = gen.generate(seed=0, **c)
    r = _run(S, T)
    assert np.isfinite(r["X"]).all() and (r["e"] <= 0).all()
    rn = oracle.tgevc(S, T, protect=False)
    assert (~np.isfinite(rn["X"]).all(axis=0)).sum() > 0


# ---- back-transformation (xTGEVC HOWMNY='B'; include/zz.h zz_tgevc_back) ----

@pytest.mark.parametrize("seed", range(5))
def test_lapack_dtgevc_back_C1(seed):
    # LAPACK's own back-transform (VR = V on entry) pins oracle.tgevc_back: the product
    # V X and the normalisation of the back-transformed columns
    _lapack_or_skip()
    S, T, _ = gen.config("C1", seed=seed)
    V = gen.orthogonal(S.shape[0], seed=seed)
    r = oracle.tgevc_back(S, T, V)
    info, VR = lapack_pin.dtgevc_back(S, T, V)
    assert info == 0 and r["status"] == 0
    lay = checks.column_layout(None, None, S)
    raw, ali = checks.parity(r["W"], VR, lay)
    assert ali.max() < 1e-11 and raw.max() < 1e-11, (ali.max(), raw.max())


def test_back_identity_V_is_the_plain_result():
    # V = I: the back-transform of the normalised X is X again, up to the renormalisation
    # (X's maximum is 1 within one rounding, R11: each entry moves by at most 2 ulps)
    S, T, _ = gen.config("C1", seed=2)
    r0 = oracle.tgevc(S, T)
    r = oracle.tgevc_back(S, T, np.eye(S.shape[0], order="F"))
    assert np.all(np.abs(r["W"] - r0["X"]) <= 4 * 2.0 ** -53 * np.abs(r0["X"]))


def test_back_residual_on_the_original_pencil():
    # A = Q S V^T, B = Q T V^T: the back-transformed W solves A W D = B W Bm
    m = 300
    S, T, _ = gen.generate(m, 45, 1.0 / m, seed=11, gap_mode=2, gap=1e-4)
    V = gen.orthogonal(m, seed=1)
    Q = gen.orthogonal(m, seed=2)
    A, B = Q @ S @ V.T, Q @ T @ V.T
    r = oracle.tgevc_back(S, T, V)
    D, Bm, lay = checks.build_DB(r["pairs"], S)
    assert checks.residual(A, B, r["W"], D, Bm) <= 10 * m * 2.0 ** -53
    # normalisation: max |w| = 1 (real), max |Re| + |Im| = 1 (pair), to one rounding
    for col, j, sz in lay:
        w = np.abs(r["W"][:, col]) if sz == 1 else np.abs(r["W"][:, col]) + np.abs(r["W"][:, col + 1])
        assert abs(w.max() - 1.0) <= 2 * 2.0 ** -53


def test_back_selected_subset_matches_full_columns():
    # a selected column's back-transform is the full solve's column (column independence)
    S, T, _ = gen.config("C1", seed=4)
    m = S.shape[0]
    V = gen.orthogonal(m, seed=4)
    full = oracle.tgevc_back(S, T, V)
    sel = np.zeros(m, np.int32)
    sel[[1, 10, 11, 50, 95]] = 1
    sub = oracle.tgevc_back(S, T, V, select=sel)
    lay_f = checks.column_layout(None, None, S)
    lay_s = checks.column_layout(None, None, S, sel)
    start = {j: col for col, j, _ in lay_f}
    for col, j, sz in lay_s:
        assert np.array_equal(sub["W"][:, col:col + sz], full["W"][:, start[j]:start[j] + sz])


# ---- left eigenvectors (LAPACK xTGEVC SIDE='L'; include/zz.h zz_tgevc_left) ----

def _left_residual(S, T, Y, lay, pairs):
    """max over columns of ||y^H (beta S - alpha T)|| / ((|beta| ||S|| + |alpha| ||T||) ||y||)"""
    worst = 0.0
    nS, nT = np.linalg.norm(S), np.linalg.norm(T)
    for col, j, sz in lay:
        y = Y[:, col] + (1j * Y[:, col + 1] if sz == 2 else 0.0)
        a, b, be = pairs[j]
        al = a + 1j * abs(b)
        r = np.conj(y) @ (be * S - al * T)
        worst = max(worst, np.linalg.norm(r) / ((abs(be) * nS + abs(al) * nT) * np.linalg.norm(y)))
    return worst


@pytest.mark.parametrize("seed", range(5))
def test_lapack_dtgevc_left_C1(seed):
    _lapack_or_skip()
    S, T, _ = gen.config("C1", seed=seed)
    r = oracle.tgevc_left(S, T)
    info, VL = lapack_pin.dtgevc_left(S, T)
    assert info == 0 and r["status"] == 0
    lay = checks.column_layout(None, None, S)
    raw, ali = checks.parity(r["Y"], VL, lay)
    assert ali.max() < 1e-11 and raw.max() < 1e-11, (ali.max(), raw.max())


def test_lapack_left_larger_zero_inf_and_subset():
    _lapack_or_skip()
    S, T, _ = gen.generate(500, 75, 1.0 / 500, seed=7, gap_mode=2, gap=1e-4, n_zero=5, n_inf=5)
    r = oracle.tgevc_left(S, T)
    info, VL = lapack_pin.dtgevc_left(S, T)
    lay = checks.column_layout(None, None, S)
    raw, ali = checks.parity(r["Y"], VL, lay)
    assert info == 0 and ali.max() < 1e-10, ali.max()
    sel = np.zeros(500, np.int32)
    sel[[0, 3, 100, 101, 250, 499]] = 1
    rs = oracle.tgevc_left(S, T, select=sel)
    info, VLs = lapack_pin.dtgevc_left(S, T, select=sel)
    lay_s = checks.column_layout(None, None, S, sel)
    raw, ali = checks.parity(rs["Y"], VLs, lay_s)
    assert info == 0 and ali.max() < 1e-10, ali.max()


def test_left_definition_zeros_and_status():
    S, T, _ = gen.config("C1", seed=6)
    r = oracle.tgevc_left(S, T)
    a, b, be, kd, st = oracle.eig_pairs(S, T)
    pairs = np.stack([a, b, be], axis=1)
    lay = checks.column_layout(None, None, S)
    assert _left_residual(S, T, r["Y"], lay, pairs) < 1e-14
    for col, j, sz in lay:     # exact zeros above the eigenvalue's block
        assert np.all(r["Y"][:j, col:col + sz] == 0.0)
    # a 2x2 block with real eigenvalues is reported by its first row in S (1-based)
    S2 = np.array([[0.5, 0.1, 0.2, 0.1], [0.0, 1.0, 0.3, 0.2], [0.0, 1.0, 1.0, 0.3], [0, 0, 0, 2.0]], order="F")
    assert oracle.tgevc_left(S2, np.eye(4, order="F"))["status"] == 2 == oracle.tgevc(S2, np.eye(4, order="F"))["status"]
