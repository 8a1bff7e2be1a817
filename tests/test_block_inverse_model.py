"""Reading R24: the in-tile solve of k_diag3 through block-local inverses
G = (beta S_bb - alpha T_bb)^-1, modelled in numpy (complex128, the GPU's row-by-row
right-looking formation of G and x = G y), agrees with the oracle's protected substitution and
has a small componentwise backward error on a C2-like pencil; and the conditioning guard
||G|| ||D|| <= 2^40 is what separates the blocks of clustered stress pencils.  Test of the
design, not of the GPU (the GPU parity tests cover the kernel)."""
import numpy as np
import pytest

import gen
import oracle
from tests import checks


def _kinds_and_blocks(S):
    m = S.shape[0]
    sub = np.r_[np.diagonal(S, -1), 0.0]
    kind = np.zeros(m, int)
    j = 0
    while j < m:
        if j + 1 < m and sub[j] != 0:
            kind[j], kind[j + 1] = 1, 2
            j += 2
        else:
            j += 1
    bs = []
    for b in range((m + 7) // 8):
        v = 8 * b
        if b > 0 and kind[v] == 2:
            v -= 1
        bs.append(v)
    bs.append(m)
    return kind, bs


def _g_rows(D, kind):
    """rows of G = D^-1, each formed right-looking as the kernel does (2x2 blocks inverted
    explicitly)"""
    n = D.shape[0]
    G = np.zeros((n, n), complex)
    for q in range(n):
        acc = np.zeros(n, complex)
        acc[q] = 1
        J = 0
        while J < n:
            if kind[J] == 1 and J + 1 < n:
                B = D[J:J + 2, J:J + 2]
                inv = np.array([[B[1, 1], -B[0, 1]], [-B[1, 0], B[0, 0]]]) / (B[0, 0] * B[1, 1] - B[0, 1] * B[1, 0])
                g = acc[J:J + 2] @ inv
                acc[J:J + 2] = g
                acc[J + 2:] -= g[0] * D[J, J + 2:] + g[1] * D[J + 1, J + 2:]
                J += 2
            else:
                acc[J] = acc[J] / D[J, J]
                acc[J + 1:] -= acc[J] * D[J, J + 1:]
                J += 1
        G[q] = acc
    return G


def _solve_column(S, T, kind, bs, j, sz, a, b, be, kappas):
    m = S.shape[0]
    al = complex(a, b)
    D = be * S - al * T
    r = j + sz - 1
    x = np.zeros(m, complex)
    if sz == 2:       # tip rule of a pair (reading R10)
        p, q = be * S[r, r - 1], D[r, r]
        if abs(p) >= abs(q.real) + abs(q.imag):
            x[r], x[r - 1] = 1, -q / p
        else:
            x[r - 1], x[r] = 1, -p / q
    else:
        x[r] = 1
    top = j
    y = -(D[:top, top:r + 1] @ x[top:r + 1])
    bi = max(i for i in range(len(bs) - 1) if bs[i] <= max(top - 1, 0))
    s0 = bs[bi]
    if top > s0:      # the tip's own block: substitution
        xb = np.linalg.solve(D[s0:top, s0:top], y[s0:top])
        x[s0:top] = xb
        y[:s0] -= D[:s0, s0:top] @ xb
    for k in range(bi - 1, -1, -1):
        s, e = bs[k], bs[k + 1]
        G = _g_rows(D[s:e, s:e], kind[s:e])
        kappas.append(np.abs(G).sum(1).max() * np.abs(D[s:e, s:e]).sum(1).max())
        xb = G @ y[s:e]
        x[s:e] = xb
        y[:s] -= D[:s, s:e] @ xb
    return x


def _model(S, T, ncols, seed=0):
    m = S.shape[0]
    kind, bs = _kinds_and_blocks(S)
    a_, b_, be_, _, _ = oracle.eig_pairs(S, T)
    ref = oracle.tgevc(S, T)
    lay = checks.column_layout(None, None, S)
    pick = sorted(np.random.default_rng(seed).choice(len(lay), min(ncols, len(lay)), replace=False))
    kappas, cols, sub_lay, worst, off = [], [], [], 0.0, 0
    for i in pick:
        col, j, sz = lay[i]
        x = _solve_column(S, T, kind, bs, j, sz, a_[j], b_[j], be_[j], kappas)
        zr = ref["X"][:, col] + (1j * ref["X"][:, col + 1] if sz == 2 else 0)
        x = x / (np.max(np.abs(x.real) + np.abs(x.imag)) if sz == 2 else np.max(np.abs(x.real)))
        ip = np.vdot(zr, x)
        worst = max(worst, np.linalg.norm(x - ip / abs(ip) * zr) / np.linalg.norm(zr))
        cols.append(x.real[:, None] if sz == 1 else np.stack([x.real, x.imag], 1))
        sub_lay.append((off, j, sz))
        off += sz
    pairs = np.stack([a_, b_, be_], 1)
    bwd = checks.comp_backward_error(S, T, np.concatenate(cols, 1), pairs, sub_lay, m)
    return worst, bwd, np.array(kappas)


def test_block_inverse_model_moderate():
    S, T, _ = gen.generate(600, 90, 1.0 / 600, seed=3, gap_mode=2, gap=1e-5)
    worst, bwd, kap = _model(S, T, 40)
    assert worst < 1e-10, worst
    assert bwd <= 10 * S.shape[0] * 2.0 ** -53, bwd
    assert np.quantile(kap, 0.99) < 2.0 ** 40      # the guard passes: the fast path is used


def test_block_inverse_guard_on_clustered_stress():
    c = dict(gen.CONFIGS["C5"])
    c.update(m=600, n2=90, stress_tile=32, stress_frac=0.0)
    S, T, _ = gen.generate(seed=0, **c)
    with np.errstate(all="ignore"):
        _, _, kap = _model(S, T, 20)
    kap = kap[np.isfinite(kap)]
    # off-diagonal N(0,1) entries and clustered eigenvalues: a share of the blocks is ill
    # conditioned enough that the guard sends them to the substitution
    assert (kap > 2.0 ** 40).any() and np.median(kap) < 2.0 ** 40
