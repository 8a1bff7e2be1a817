"""Pins of the oracle's eigenvalue pairs (alpha, beta): closed forms
for 1x1 blocks and for the generator's 2x2 blocks, SPEC examples S:64-66, and the
assumption-2 error code."""
import numpy as np
import pytest

import gen
import oracle


def test_1x1_exact_ratio_and_sign():
    S = np.array([[2.0, 0.3, -1.0], [0, 3.0, 0.2], [0, 0, -0.75]], order="F")
    T = np.array([[1.0, 0.5, 0.1], [0, 0.0, 0.4], [0, 0, -0.5]], order="F")
    a, b, be, kd, st = oracle.eig_pairs(S, T)
    assert st == 0
    assert np.all(b == 0) and np.all(kd == 0)
    # (2,1) up to a power of two; S:65 infinite eigenvalue (3, 0)
    assert a[0] / be[0] == 2.0
    assert be[1] == 0.0 and a[1] > 0
    # negative T diagonal: both signs flipped, beta >= 0
    assert be[2] > 0 and a[2] / be[2] == (-0.75) / (-0.5)
    for j in range(3):
        mx = max(be[j], abs(a[j]) + abs(b[j]))
        assert 0.5 <= mx < 1.0
        # exact power-of-two multiple of (S_jj, |T_jj|)
        k = np.log2(abs(a[j]) / abs(S[j, j]))
        assert k == np.round(k)


def test_indefinite_kind():
    S = np.array([[0.0, 1.0], [0.0, 2.0]], order="F")
    T = np.array([[0.0, 1.0], [0.0, 1.0]], order="F")
    a, b, be, kd, st = oracle.eig_pairs(S, T)
    assert st == 0 and kd[0] == 2 and kd[1] == 0


def test_spec_rotation_block():
    # S=[[0,1],[-1,0]], T=I -> (alpha, beta) = (i, 1) up to scale
    S = np.array([[0.0, 1.0], [-1.0, 0.0]], order="F")
    T = np.eye(2, order="F")
    a, b, be, kd, st = oracle.eig_pairs(S, T)
    assert st == 0 and kd[0] == 1 and kd[1] == 1
    assert a[0] == 0.0 and b[0] > 0 and b[0] / be[0] == 1.0


def test_real_2x2_block_is_error():
    # S=[[1,0],[1,1]], T=I has the real double eigenvalue 1 -> INFO = 1 (1-based)
    S = np.array([[5.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 1.0, 1.0]], order="F")
    T = np.eye(3, order="F")
    *_, st = oracle.eig_pairs(S, T)
    assert st == 2


@pytest.mark.parametrize("seed", range(4))
def test_generator_blocks_closed_form(seed):
    # generator 2x2 block [[a,b],[-c,a t2/t1]], diag(t1,t2): lambda = a/t1 +- i sqrt(bc/(t1 t2))
    S, T, lam = gen.config("C1", seed=seed)
    a, b, be, kd, st = oracle.eig_pairs(S, T)
    assert st == 0
    got = (a + 1j * b) / be
    for j in range(S.shape[0]):
        if kd[j] == 1:
            ref = lam[j] if lam[j].imag > 0 else np.conj(lam[j])
            assert abs(got[j] - ref) <= 1e-14 * abs(ref)
        else:
            assert a[j] / be[j] == S[j, j] / T[j, j]
