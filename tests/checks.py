"""Verification helpers shared by the test files (test code only; no product logic).

* residual(): the normwise relative residual of BASELINE.json north_star / DESIGN.md R7,
  ||S X D - T X B||_F / ((||S||_F ||D||_2 + ||T||_F ||B||_2) ||X||_F).
* comp_backward_error(): per-column componentwise backward error (strong check).
* parity(): per-column relative 2-norm difference, raw and phase-aligned for pairs.
* brute_null_vector(): long-double complete-pivoting Gaussian elimination of the full
  complex matrix beta S - alpha T (independent of the triangular structure).
"""
import numpy as np

U = 2.0 ** -53


def column_layout(pairs_a, pairs_b, S, select=None):
    """List of (first_col, row_of_block_first, block_size, kind) in packed order, computed
    from the structure of S (subdiagonal) and b != 0 for pairs."""
    m = S.shape[0]
    out = []
    j = 0
    col = 0
    while j < m:
        two = j + 1 < m and S[j + 1, j] != 0.0
        sz = 2 if two else 1
        sel = select is None or select[j] or (two and select[j + 1])
        if sel:
            out.append((col, j, sz))
            col += sz
        j += sz
    return out


def build_DB(pairs, S, select=None):
    """D (n) and B (n x n block diagonal) of PAPER.md:83-99 for the packed columns, from
    per-row normalised pairs (a, b, beta)."""
    lay = column_layout(pairs[:, 0], pairs[:, 1], S, select)
    n = sum(sz for _, _, sz in lay)
    D = np.zeros(n)
    B = np.zeros((n, n))
    for col, j, sz in lay:
        a, b, be = pairs[j]
        if sz == 1:
            D[col] = be
            B[col, col] = a
        else:
            D[col:col + 2] = be
            B[col:col + 2, col:col + 2] = [[a, b], [-b, a]]
    return D, B, lay


def residual(S, T, X, D, B):
    """normwise relative residual; accumulation in float64 (or long double if small)"""
    if S.shape[0] <= 300:
        Sl, Tl, Xl = (np.asarray(A, dtype=np.longdouble) for A in (S, T, X))
        R = (Sl @ Xl) * np.asarray(D, dtype=np.longdouble) - (Tl @ Xl) @ np.asarray(B, dtype=np.longdouble)
        num = float(np.sqrt((R * R).sum()))
    else:
        R = (S @ X) * D - (T @ X) @ B
        num = float(np.linalg.norm(R))
    nd = float(np.max(np.abs(D))) if D.size else 0.0
    nb = float(np.linalg.norm(B, 2)) if B.size else 0.0
    den = (np.linalg.norm(S) * nd + np.linalg.norm(T) * nb) * np.linalg.norm(X)
    return num / den if den > 0 else 0.0


def to_complex(X, lay):
    """list of complex eigenvectors z (one per block) from packed real columns"""
    out = []
    for col, j, sz in lay:
        if sz == 1:
            out.append(X[:, col].astype(complex))
        else:
            out.append(X[:, col] + 1j * X[:, col + 1])
    return out


def parity(Xa, Xb, lay):
    """per-block (raw, phase_aligned) relative 2-norm differences of Xa vs reference Xb"""
    raw, ali = [], []
    for za, zb in zip(to_complex(Xa, lay), to_complex(Xb, lay)):
        nb = np.linalg.norm(zb)
        raw.append(np.linalg.norm(za - zb) / nb)
        ip = np.vdot(zb, za)
        c = ip / abs(ip) if abs(ip) > 0 else 1.0
        ali.append(np.linalg.norm(za - c * zb) / nb)
    return np.array(raw), np.array(ali)


def comp_backward_error(S, T, X, pairs, lay, m):
    """max over columns of omega_c = max_i |(beta S z - alpha T z)_i| /
    (beta (|S||z|)_i + |alpha| (|T||z|)_i), rows with tiny denominators excluded."""
    aS, aT = np.abs(S), np.abs(T)
    nS, nT = np.abs(S).sum(axis=1).max(), np.abs(T).sum(axis=1).max()
    worst = 0.0
    for z, (col, j, sz) in zip(to_complex(X, lay), lay):
        a, b, be = pairs[j]
        al = complex(a, b)
        r = be * (S @ z) - al * (T @ z)
        den = be * (aS @ np.abs(z)) + abs(al) * (aT @ np.abs(z))
        thr = 2.0 ** -1021 * (be * nS + abs(al) * nT)
        ok = den >= thr
        if ok.any():
            worst = max(worst, float(np.max(np.abs(r[ok]) / den[ok])))
    return worst


def brute_null_vector(S, T, a, b, beta):
    """Null vector of M = beta S - alpha T (complex, long double) by complete-pivoting
    Gaussian elimination of the FULL matrix; the free variable is set to 1.  Returned
    normalised so that max(|Re|+|Im|) = 1 (LAPACK convention, phase arbitrary)."""
    m = S.shape[0]
    al = np.clongdouble(complex(a, b))
    M = np.asarray(S, dtype=np.clongdouble) * np.longdouble(beta) - al * np.asarray(T, dtype=np.clongdouble)
    colperm = np.arange(m)
    for k in range(m - 1):
        sub = np.abs(M[k:, k:])
        i, j = np.unravel_index(np.argmax(sub), sub.shape)
        i += k
        j += k
        M[[k, i], :] = M[[i, k], :]
        M[:, [k, j]] = M[:, [j, k]]
        colperm[[k, j]] = colperm[[j, k]]
        if M[k, k] == 0:
            continue
        l = M[k + 1:, k] / M[k, k]
        M[k + 1:, k:] -= np.outer(l, M[k, k:])
    # back substitution with the last (near-zero pivot) variable set to 1
    y = np.zeros(m, dtype=np.clongdouble)
    y[m - 1] = 1
    for k in range(m - 2, -1, -1):
        y[k] = -(M[k, k + 1:] @ y[k + 1:]) / M[k, k]
    z = np.zeros(m, dtype=np.clongdouble)
    z[colperm] = y
    nrm = np.max(np.abs(z.real) + np.abs(z.imag))
    return (z / nrm).astype(complex)
