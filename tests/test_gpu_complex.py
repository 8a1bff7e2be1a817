"""GPU parity of zz_ztgevc (complex pencils) against the complex
oracle (oracle/zz_oracle_z.c), through the C ABI binding.

Tolerance: both sides normalise to max(|Re|+|Im|) = 1 from a real positive tip, so the
columns are unique and compared entrywise.  The GPU sums the update in a different order
(ZGEMM), so entries differ by rounding amplified by the conditioning of the substitution:
for these pencils (off-diagonals N(0, 1/m), separated eigenvalues) 1e-10 absolute is
> 1000 x the observed difference and far below any algorithmic error (a dropped term or
a wrong sign moves entries by O(1e-3) or more)."""
import numpy as np
import pytest

import gen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def zz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_04776_b200 as zz
    zz.init(0)
    yield zz
    zz.set_tile(0)


def _dev(A):
    return torch.from_numpy(np.asfortranarray(A)).cuda().t().contiguous().t()


def _run(zz, S, T, select=None, tile=0):
    zz.set_tile(tile)
    try:
        X, e = zz.ztgevc(_dev(S), _dev(T), select=select)
        torch.cuda.synchronize()
    finally:
        zz.set_tile(0)
    return X.cpu().numpy(), e.cpu().numpy()


@pytest.mark.parametrize("m,tile,seed", [(1, 32, 0), (31, 32, 1), (96, 32, 2), (200, 64, 3), (777, 64, 4),
                                         (333, 48, 5)])
def test_ztgevc_parity(zz, m, tile, seed):
    S, T = gen.complex_pencil(m, seed=seed)
    X, e = _run(zz, S, T, tile=tile)
    ref = oracle.ztgevc(S, T)
    assert ref["status"] == 0
    assert X.shape == ref["X"].shape
    assert np.array_equal(np.tril(X, -1), np.zeros_like(X))       # zeros below the tip
    err = np.abs(X - ref["X"]).max()
    assert err < TOL, err
    assert zz.last_info()["n_tiles"] == (m + tile - 1) // tile


def test_ztgevc_select(zz):
    m = 500
    S, T = gen.complex_pencil(m, seed=7)
    sel = np.zeros(m, np.int32)
    sel[[0, 1, 63, 64, 65, 200, 498, 499]] = 1
    X, _ = _run(zz, S, T, select=sel)
    ref = oracle.ztgevc(S, T, select=sel)
    assert X.shape == (m, 8)
    assert np.abs(X - ref["X"]).max() < TOL


def test_ztgevc_stress_scaling(zz):
    """Off-diagonals of 1e150 in alternate rows: the unprotected substitution overflows;
    the robust path scales (col_scale_exp < 0) and matches the oracle after normalisation."""
    m = 160
    S, T = gen.complex_pencil(m, seed=4, stress=True)
    X, e = _run(zz, S, T, tile=32)
    ref = oracle.ztgevc(S, T)
    assert np.isfinite(X).all()
    assert (e < 0).any()
    big = np.abs(ref["X"]) > 1e-200
    assert np.abs(X[big] - ref["X"][big]).max() < 1e-9
    assert np.abs(X[~big]).max() < 1e-190


def test_ztgevc_indefinite_and_infinite(zz):
    m = 70
    S, T = gen.complex_pencil(m, seed=8)
    S[10, 10] = 0.0
    T[10, 10] = 0.0          # indefinite: e_10
    T[40, 40] = 0.0          # infinite eigenvalue
    X, _ = _run(zz, S, T, tile=32)
    ref = oracle.ztgevc(S, T)
    assert ref["stats"][2] == 1
    assert np.array_equal(X[:, 10], np.eye(m)[:, 10])
    assert np.abs(X - ref["X"]).max() < TOL


def test_ztgevc_status(zz):
    S, T = gen.complex_pencil(50, seed=9)
    T2 = T.copy()
    T2[20, 20] += 1e-3j
    with pytest.raises(zz.ZZError) as ei:
        _run(zz, S, T2)
    assert ei.value.status == -107
    S2 = S.copy()
    S2[5, 5] = np.inf
    with pytest.raises(zz.ZZError) as ei:
        _run(zz, S2, T2)
    assert ei.value.status == -104          # row 5 comes first
    X, _ = _run(zz, S[:0, :0], T[:0, :0])
    assert X.shape == (0, 0)


@pytest.mark.parametrize("m", [4000, 6000])
def test_ztgevc_large_sampled(zz, m):
    """m = 4000 and 6000 in the bench launch configuration (tile 64, the library's default
    step groups): sampled columns against the oracle's selected-column solve.  At m = 6000
    the steps with more than 148 x 32 active columns run k_zdiag with four columns per warp,
    the others with two."""
    S, T = gen.complex_pencil(m, seed=10)
    X, _ = _run(zz, S, T)
    cols = sorted([0, 1, 999, 2047, 2048, 3071, m // 2 + 5, m - 1003, m - 2, m - 1])
    sel = np.zeros(m, np.int32)
    sel[cols] = 1
    ref = oracle.ztgevc(S, T, select=sel)
    assert np.abs(X[:, cols] - ref["X"]).max() < TOL


def _run_mode(zz, S, T, la, fusion, select=None, tile=64):
    zz.set_lookahead(la)
    zz.set_fusion(fusion)
    try:
        return _run(zz, S, T, select=select, tile=tile)
    finally:
        zz.set_lookahead(1)
        zz.set_fusion(0)


@pytest.mark.parametrize("fusion", [1, 2, 3, 4])
@pytest.mark.parametrize("la", [0, 1])
@pytest.mark.parametrize("stress", [False, True])
def test_ztgevc_lookahead_and_step_groups(zz, la, fusion, stress):
    """Both schedules (zz_set_lookahead: the chain of a step group on a high-priority stream
    beside the rest of the previous group's update, or everything in stream order) and step
    groups of 1-4 tiles (zz_set_fusion: one update with K segments per group) against the
    oracle, on a pencil with selected columns opening mid-wavefront and mid-group."""
    m = 700
    S, T = gen.complex_pencil(m, seed=12, stress=stress)
    sel = np.ones(m, np.int32)
    sel[600:] = 0            # the top steps have no active columns
    sel[::7] = 0
    X, e = _run_mode(zz, S, T, la, fusion, select=sel, tile=64)
    info = zz.last_info()
    ref = oracle.ztgevc(S, T, select=sel)
    assert np.isfinite(X).all()
    big = np.abs(ref["X"]) > 1e-200
    assert np.abs(X[big] - ref["X"][big]).max() < (1e-9 if stress else TOL)
    if stress:
        assert (e < 0).any()
    assert (info["fused_pairs"] > 0) == (fusion > 1)


@pytest.mark.parametrize("fusion", [1, 4])
def test_ztgevc_schedule_and_select_bitwise(zz, fusion):
    """The lookahead only reorders launches over disjoint rows, and a column's arithmetic does
    not depend on which other columns are selected (step groups are fixed by the tile index):
    bit for bit the same columns (stress pencil: scalings inside the groups)."""
    m = 640
    S, T = gen.complex_pencil(m, seed=14, stress=True)
    X0, e0 = _run_mode(zz, S, T, 0, fusion, tile=64)
    X1, e1 = _run_mode(zz, S, T, 1, fusion, tile=64)
    assert np.array_equal(X0, X1) and np.array_equal(e0, e1)
    assert (e0 < 0).any()
    sel = np.zeros(m, np.int32)
    cols = [3, 64, 200, 201, 350, 511, 512, 639]
    sel[cols] = 1
    Xs, es = _run_mode(zz, S, T, 1, fusion, select=sel, tile=64)
    assert np.array_equal(Xs, X0[:, cols]) and np.array_equal(es, e0[cols])


def test_ztgevc_padded_leading_dimensions(zz):
    """lds, ldt, ldx larger than m (sub-views of bigger column-major buffers): the same
    columns as the packed call, and the padding rows of X are not written."""
    m = 150
    S, T = gen.complex_pencil(m, seed=13)
    X0, _ = _run(zz, S, T, tile=32)

    def padded(A, extra):
        B = torch.zeros((A.shape[1], m + extra), dtype=torch.complex128, device="cuda").t()
        B[:m] = torch.from_numpy(A).cuda()
        return B[:m]

    Sd, Td = padded(S, 5), padded(T, 3)
    Xbuf = torch.full((m, m + 7), 7.0 + 7.0j, dtype=torch.complex128, device="cuda").t()
    zz.set_tile(32)
    try:
        zz.ztgevc(Sd, Td, X=Xbuf[:m])
        torch.cuda.synchronize()
    finally:
        zz.set_tile(0)
    Xp = Xbuf.cpu().numpy()
    assert np.array_equal(Xp[:m], X0)
    assert (Xp[m:] == 7.0 + 7.0j).all()
