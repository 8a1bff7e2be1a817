"""GPU parity tests (-m gpu): the CUDA path through the C ABI against the oracle on the
same seeded inputs, plus invariants, edge cases, error codes, the scaling path and the
full-size configurations in the launch configuration bench.py times.

Tolerances: BASELINE.json north_star fixes the bar: every normalised column within 1e-10
relative 2-norm of the oracle (phase-aligned for pairs; raw as well since both sides use
the tip rule of reading R10) on the moderate-growth configs, and the normwise residual
<= 10 m 2^-53 (reading R7).  Bitwise equality is required where the arithmetic is
identical by construction (column independence / sharding, leading dimensions,
power-of-two equivariance)."""
import numpy as np
import pytest

import gen
import oracle
from tests import checks

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
U = 2.0 ** -53
TOL = 1e-10


@pytest.fixture(scope="module")
def zz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_04776_b200 as zz
    zz.init(0)
    yield zz
    zz.set_tile(0)


def to_dev(A, ld=None):
    m, n = A.shape
    ld = ld or m
    buf = torch.zeros((max(n, 1), ld), dtype=torch.float64, device="cuda")
    buf[:n, :m] = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    return buf.t()[:m, :n]


def solve(zz, S, T, mb=0, select=None, lds=None, ldx=None, Sd=None, Td=None):
    zz.set_tile(mb)
    m = S.shape[0] if S is not None else Sd.shape[0]
    if Sd is None:
        Sd, Td = to_dev(S, lds), to_dev(T, lds)
    n = oracle.count_columns(S, select) if S is not None else m
    X = None
    if ldx is not None:
        X = torch.full((max(n, 1), ldx), np.nan, dtype=torch.float64, device="cuda").t()[:m, :n]
    X, e = zz.tgevc(Sd, Td, select=select, X=X, n_sel=n)
    torch.cuda.synchronize()
    info = zz.last_info()
    info["views"] = zz.last_views()
    return X.cpu().numpy(), e.cpu().numpy(), info


def check_logmax_and_pairs(S, views, ref, select=None, pairs_bitwise=True):
    """the GPU's L_c = log2(max measure of the tip-normalised vector)
    (include/zz.h zz_info_t.d_logmax; Definition 1) within 1e-10 relative
    of the oracle's, and the normalised eigenvalue pairs the pivots were formed with
    bitwise equal to the oracle's (reading R17)."""
    lay = checks.column_layout(None, None, S, select)
    L = views["logmax"]
    assert L is not None and L.shape == ref["logmax"].shape
    dL = np.abs(L - ref["logmax"]) / np.maximum(1.0, np.abs(ref["logmax"]))
    assert np.isfinite(L).all() and dL.max() <= TOL, (dL.max(), int(np.argmax(dL)))
    if pairs_bitwise:
        for col, j, sz in lay:
            for k in range(sz):
                got = (views["a"][col + k], views["b"][col + k], views["beta"][col + k])
                assert got == tuple(ref["pairs"][j]), (col, j, got, ref["pairs"][j])
    return dL.max()


def check_against_oracle(S, T, X, e, select=None, tol=TOL, ref=None, info=None):
    ref = ref or oracle.tgevc(S, T, select=select)
    assert ref["status"] == 0
    if info is not None and info.get("views") is not None:
        check_logmax_and_pairs(S, info["views"], ref, select, pairs_bitwise=not info["prescaled"])
    lay = checks.column_layout(None, None, S, select)
    raw, ali = checks.parity(X, ref["X"], lay)
    assert np.isfinite(X).all()
    assert ali.max() <= tol, (ali.max(), int(np.argmax(ali)))
    assert raw.max() <= tol, (raw.max(), int(np.argmax(raw)))
    # invariants: e <= 0, equal pair exponents, exact zeros below, LAPACK normalisation
    assert (e <= 0).all()
    for col, j, sz in lay:
        assert np.all(X[j + sz:, col:col + sz] == 0.0)
        if sz == 2:
            assert e[col] == e[col + 1]
            mx = np.max(np.abs(X[:, col]) + np.abs(X[:, col + 1]))
        else:
            mx = np.max(np.abs(X[:, col]))
        assert abs(mx - 1.0) <= 4 * U
    D, B, _ = checks.build_DB(ref["pairs"], S, select)
    if S.shape[0] <= 3000:
        res = checks.residual(S, T, X, D, B)
        assert res <= 10 * S.shape[0] * U, res
    return ref, raw, ali


@pytest.mark.parametrize("seed", range(10))
def test_C1_parity(zz, seed):
    S, T, _ = gen.config("C1", seed=seed)
    X, e, info = solve(zz, S, T, mb=32)
    assert info["n_tiles"] >= 3
    check_against_oracle(S, T, X, e, info=info)


@pytest.mark.parametrize("mb", [32, 64, 96, 128, 160])
def test_C2_parity_tile_sweep(zz, mb):
    S, T, _ = gen.config("C2", seed=0)
    X, e, info = solve(zz, S, T, mb=mb)
    check_against_oracle(S, T, X, e, info=info)


@pytest.mark.parametrize("m", [1, 2, 3, 5, 31, 33, 65, 130, 257, 511, 1025])
def test_ragged_sizes(zz, m):
    n2 = (3 * m) // 20
    S, T, _ = gen.generate(m, n2, 1.0 / m, seed=m, gap_mode=2, gap=1e-4)
    for mb in (32, 48, 160):
        X, e, info = solve(zz, S, T, mb=mb)
        check_against_oracle(S, T, X, e, info=info)


def test_all_pairs_and_all_real(zz):
    for m, n2 in [(64, 32), (66, 33), (100, 0)]:
        S, T, _ = gen.generate(m, n2, 1.0 / m, seed=7, gap_mode=2, gap=1e-4)
        X, e, info = solve(zz, S, T, mb=32)
        check_against_oracle(S, T, X, e, info=info)


def test_zero_infinite_indefinite_negative(zz):
    S, T, _ = gen.generate(300, 45, 1.0 / 300, seed=11, gap_mode=2, gap=1e-4, n_zero=4, n_inf=5)
    # a negative T diagonal entry and an indefinite 1x1 block
    d = [j for j in range(1, 299) if S[j, j - 1] == 0 and S[j + 1, j] == 0 and T[j, j] != 0]
    T[d[3], d[3]] *= -1
    S[d[7], d[7]] = 0.0
    T[d[7], d[7]] = 0.0
    X, e, info = solve(zz, S, T, mb=64)
    assert info["n_indefinite"] == 1
    check_against_oracle(S, T, X, e, info=info)
    assert np.array_equal(X[:, d[7]], np.eye(300)[:, d[7]])


def test_error_codes(zz):
    # 2x2 block with real eigenvalues -> +j (1-based first row), as DTGEVC
    S = np.array([[0.5, 0.1, 0.2, 0.1], [0.0, 1.0, 0.3, 0.2], [0.0, 1.0, 1.0, 0.3], [0, 0, 0, 2.0]], order="F")
    T = np.eye(4, order="F")
    with pytest.raises(zz.ZZError) as ei:
        solve(zz, S, T, mb=32)
    assert ei.value.status == 2 == oracle.tgevc(S, T)["status"]
    # overlapping 2x2 blocks -> -105
    S2 = S.copy()
    S2[3, 2] = 1.0
    with pytest.raises(zz.ZZError) as ei:
        solve(zz, S2, T, mb=32)
    assert ei.value.status == -105
    # non-finite diagonal block -> -104
    S3 = np.triu(S)
    S3[1, 1] = np.inf
    with pytest.raises(zz.ZZError) as ei:
        solve(zz, S3, T, mb=32)
    assert ei.value.status == -104


def test_set_fusion_arguments(zz):
    lib = zz.load()
    assert lib.zz_set_fusion(-1) == -1 and lib.zz_set_fusion(7) == -1 and lib.zz_set_fusion(0) == 0
    for k in (1, 6, 4):
        assert lib.zz_set_fusion(k) == 0
    assert lib.zz_set_fusion(0) == 0   # back to the library defaults


def test_select_subsets_bitwise(zz):
    S, T, _ = gen.config("C2", seed=1)
    m = S.shape[0]
    Xf, ef, _ = solve(zz, S, T, mb=64)
    lay = checks.column_layout(None, None, S)
    rng = np.random.default_rng(5)
    for frac in (0.001, 0.05, 0.5):
        sel = (rng.random(m) < frac).astype(np.int32)
        Xs, es, _ = solve(zz, S, T, mb=64, select=sel)
        cols = [c for (c, j, sz) in lay if sel[j] or (sz == 2 and sel[j + 1]) for c in range(c, c + sz)]
        assert np.array_equal(Xs, Xf[:, cols])
        assert np.array_equal(es, ef[cols])
    # empty selection
    Xs, es, info = solve(zz, S, T, mb=64, select=np.zeros(m, np.int32))
    assert Xs.shape == (m, 0) and info["n_sel"] == 0


def test_leading_dimensions_and_alignment(zz):
    S, T, _ = gen.config("C2", seed=0, m=700, n2=105)
    X0, e0, _ = solve(zz, S, T, mb=64)
    for lds, ldx in [(701, 703), (704, 700), (1001, 1001)]:
        X1, e1, _ = solve(zz, S, T, mb=64, lds=lds, ldx=ldx)
        assert np.array_equal(X1, X0) and np.array_equal(e1, e0)


def test_repeat_bitwise_fused_pairs(zz):
    # full 128-row tiles: every grouped update runs K = 3 x 256 (48 pipeline chunks); repeated
    # solves and an odd ldx (internal aligned workspace) must give identical bits -- this is
    # the regression test of the stage-release race of the update pipeline (DESIGN.md s.6)
    S, T, _ = gen.config("C3", seed=1, m=3000, n2=450)
    X0, e0, info = solve(zz, S, T, mb=128)
    assert info["n_tiles"] >= 20 and info["fused_pairs"] >= 6
    for _ in range(3):
        X1, e1, _ = solve(zz, S, T, mb=128)
        assert np.array_equal(X1, X0) and np.array_equal(e1, e0)
    X2, e2, _ = solve(zz, S, T, mb=128, ldx=3001)
    assert np.array_equal(X2, X0) and np.array_equal(e2, e0)


def test_power_of_two_equivariance_and_prescale(zz):
    S, T, _ = gen.config("C1", seed=6)
    X0, e0, _ = solve(zz, S, T, mb=32)
    for k in (-300, -5, 7, 200):
        X1, e1, info = solve(zz, np.ldexp(S, k), np.ldexp(T, k), mb=32)
        assert np.array_equal(X1, X0)
    # entries near Omega/4: the pre-scale path (reading R6) must trigger and change nothing
    X2, e2, info = solve(zz, np.ldexp(S, 1021), np.ldexp(T, 1021), mb=32)
    assert info["prescaled"] == 1
    assert np.array_equal(X2, X0)


def _stress(m, seed, tile=32):
    c = dict(gen.CONFIGS["C5"])
    c.update(m=m, n2=(3 * m) // 20, stress_tile=tile)
    return gen.generate(seed=seed, **c)[:2]


@pytest.mark.parametrize("m,mb", [(1000, 64), (2000, 128)])
def test_stress_scaling_path(zz, m, mb):
    S, T = _stress(m, 0)
    X, e, info = solve(zz, S, T, mb=mb)
    ref = oracle.tgevc(S, T)
    naive = oracle.tgevc(S, T, protect=False)
    n_bad = int((~np.isfinite(naive["X"]).all(axis=0)).sum())
    assert n_bad > 0                       # unprotected substitution overflows
    assert np.isfinite(X).all()            # the robust GPU path does not
    assert info["n_scaled"] > 0 and (e <= 0).all() and info["min_exp"] < 0
    # the exponents are implementation-defined; L_c = log2 |tip-normalised max| is not
    dl = check_logmax_and_pairs(S, info["views"], ref)
    print("stress m=%d: %d columns scaled, max rel |dL_c| %.2e" % (m, info["n_scaled"], dl))
    lay = checks.column_layout(None, None, S)
    for col, j, sz in lay:
        if sz == 2:
            assert e[col] == e[col + 1]
        assert np.all(X[j + sz:, col:col + sz] == 0.0)
    w = checks.comp_backward_error(S, T, X, ref["pairs"], lay, m)
    assert w <= 10 * m * U, w
    D, B, _ = checks.build_DB(ref["pairs"], S)
    assert checks.residual(S, T, X, D, B) <= 10 * m * U


def _gpu_residual(Sd, Td, Xd, pairs, S_sub, cols=None):
    """normwise residual (R7) on the GPU with FP64 GEMMs, for the column subset `cols`
    (sorted; both columns of a pair present)"""
    m = Sd.shape[0]
    lay = checks.column_layout(None, None, S_sub)
    D = np.zeros(m)
    A = np.zeros(m)
    Bc = np.zeros(m)
    kind = np.zeros(m, int)          # 0 real, 1 first of pair, 2 second
    for col, j, sz in lay:
        a, b, be = pairs[j]
        D[col:col + sz] = be
        A[col:col + sz] = a
        Bc[col:col + sz] = b
        if sz == 2:
            kind[col], kind[col + 1] = 1, 2
    cols = np.arange(m) if cols is None else np.asarray(cols)
    dev = "cuda"
    Xc = Xd[:, torch.as_tensor(cols, device=dev)]
    TX = Td @ Xc
    R = (Sd @ Xc) * torch.as_tensor(D[cols], device=dev)
    kc = kind[cols]
    a_ = torch.as_tensor(A[cols], device=dev)
    b_ = torch.as_tensor(Bc[cols], device=dev)
    nxt = torch.as_tensor(np.minimum(np.arange(len(cols)) + 1, len(cols) - 1), device=dev)
    prv = torch.as_tensor(np.maximum(np.arange(len(cols)) - 1, 0), device=dev)
    first = torch.as_tensor(kc == 1, device=dev)
    second = torch.as_tensor(kc == 2, device=dev)
    XB = a_ * TX
    XB = XB - torch.where(first, b_, torch.zeros_like(b_)) * TX[:, nxt]
    XB = XB + torch.where(second, b_, torch.zeros_like(b_)) * TX[:, prv]
    R = R - XB
    num = torch.linalg.norm(R).item()
    ab = np.hypot(A, Bc)
    den = (torch.linalg.norm(Sd).item() * D.max() + torch.linalg.norm(Td).item() * ab.max()) * \
        torch.linalg.norm(Xc).item()
    return num / den


@pytest.mark.slow
def test_C3_full_parity(zz):
    S, T, _ = gen.config("C3", seed=0)
    Sd, Td = to_dev(S), to_dev(T)
    zz.set_tile(128)
    Xd, ed = zz.tgevc(Sd, Td)
    torch.cuda.synchronize()
    views = zz.last_views()
    X, e = Xd.cpu().numpy(), ed.cpu().numpy()
    ref = oracle.tgevc(S, T)
    lay = checks.column_layout(None, None, S)
    raw, ali = checks.parity(X, ref["X"], lay)
    assert np.isfinite(X).all() and (e <= 0).all()
    assert ali.max() <= TOL and raw.max() <= TOL, (raw.max(), ali.max())
    check_logmax_and_pairs(S, views, ref)
    assert _gpu_residual(Sd, Td, Xd, ref["pairs"], S) <= 10 * S.shape[0] * U


@pytest.mark.slow
def test_C5_stress_full(zz):
    S, T, _ = gen.config("C5", seed=0)
    m = S.shape[0]
    Sd, Td = to_dev(S), to_dev(T)
    zz.set_tile(128)
    Xd, ed = zz.tgevc(Sd, Td)
    torch.cuda.synchronize()
    info = zz.last_info()
    views = zz.last_views()
    X, e = Xd.cpu().numpy(), ed.cpu().numpy()
    assert np.isfinite(X).all() and (e <= 0).all()
    # most columns scaled: the L_c agreement pins the exponents; the oracle
    # runs once (column independent, all host cores)
    assert (e < 0).mean() > 0.5
    ref = oracle.tgevc(S, T)
    assert ref["status"] == 0
    check_logmax_and_pairs(S, views, ref)
    lay = checks.column_layout(None, None, S)
    for col, j, sz in lay:
        if sz == 2:
            assert e[col] == e[col + 1]
    a, b, be, kd, st = oracle.eig_pairs(S, T)
    pairs = np.stack([a, b, be], axis=1)
    assert _gpu_residual(Sd, Td, Xd, pairs, S) <= 10 * m * U
    # componentwise backward error on a sample of columns
    rng = np.random.default_rng(0)
    pick = sorted(rng.choice(len(lay), 60, replace=False))
    sub_lay = [lay[i] for i in pick]
    cols = [c for (c, j, sz) in sub_lay for c in range(c, c + sz)]
    Xs = X[:, cols]
    lay2, off = [], 0
    for (c, j, sz) in sub_lay:
        lay2.append((off, j, sz))
        off += sz
    assert checks.comp_backward_error(S, T, Xs, pairs, lay2, m) <= 10 * m * U


@pytest.mark.slow
def test_C4_full_size_sampled(zz):
    """m = 40000 in the launch configuration bench.py times (mb = 128, all eigenvectors);
    sampled columns against the oracle computed one by one."""
    m = gen.CONFIGS["C4"]["m"]
    Sd = torch.empty((m, m), dtype=torch.float64).pin_memory().t()
    Td = torch.empty((m, m), dtype=torch.float64).pin_memory().t()
    gen.config("C4", seed=0, out=(Sd.data_ptr(), Td.data_ptr()))
    S, T = Sd.numpy(), Td.numpy()
    Sg = torch.empty((m, m), dtype=torch.float64, device="cuda").t()
    Tg = torch.empty((m, m), dtype=torch.float64, device="cuda").t()
    Sg.copy_(Sd)
    Tg.copy_(Td)
    zz.set_tile(128)
    Xd, ed = zz.tgevc(Sg, Tg)
    torch.cuda.synchronize()
    sub = np.diagonal(S, -1)
    blocks = []
    j = 0
    while j < m:
        sz = 2 if (j + 1 < m and sub[j] != 0) else 1
        blocks.append((j, sz))
        j += sz
    rng = np.random.default_rng(1)
    idx = sorted(set(rng.choice(len(blocks), 20, replace=False).tolist()) | {0, len(blocks) - 1})
    sel = np.zeros(m, np.int32)
    for b in idx:
        jj, sz = blocks[b]
        sel[jj:jj + sz] = 1
    ref = oracle.tgevc(S, T, select=sel)
    cols = np.flatnonzero(sel)
    Xg = Xd[:, torch.as_tensor(cols, device="cuda")].cpu().numpy()
    lay = checks.column_layout(None, None, S, sel)
    raw, ali = checks.parity(Xg, ref["X"], lay)
    assert np.isfinite(Xg).all()
    assert ali.max() <= TOL and raw.max() <= TOL, (raw.max(), ali.max())
    assert (ed.cpu().numpy() <= 0).all()
    assert _gpu_residual(Sg, Tg, Xd, ref["pairs"], S, cols=cols) <= 10 * m * U


def _host_solve(zz, S, T, mb, select=None, ldx=None):
    """zz_tgevc_host: host S, T, X (the end-to-end path bench.py times)"""
    zz.set_tile(mb)
    m = S.shape[0]
    n = oracle.count_columns(S, select)
    X = np.full((ldx or m, max(n, 1)), np.nan, order="F")[:m, :n]
    e = np.zeros(max(n, 1), np.int32)[:n]
    zz.tgevc_host(S, T, select=select, X=X, col_scale_exp=e)
    return X, e, zz.last_info()


@pytest.mark.parametrize("name,seed,mb", [("C1", 0, 32), ("C1", 4, 64), ("C2", 1, 128), ("C2", 2, 64)])
def test_host_path_bitwise_equal_to_device_path(zz, name, seed, mb):
    """The host-staged path (panels copied in consumption order, overlapped with the solve)
    computes exactly the device path's arithmetic."""
    S, T, _ = gen.config(name, seed=seed)
    X0, e0, i0 = solve(zz, S, T, mb=mb)
    X1, e1, i1 = _host_solve(zz, S, T, mb)
    assert np.array_equal(X1, X0) and np.array_equal(e1, e0)
    assert i1["n_tiles"] == i0["n_tiles"]
    check_against_oracle(S, T, X1, e1)


def test_host_path_select_ld_errors_and_prescale(zz):
    S, T, _ = gen.config("C2", seed=0, m=700, n2=105)
    rng = np.random.default_rng(3)
    sel = (rng.random(700) < 0.2).astype(np.int32)
    X0, e0, _ = solve(zz, S, T, mb=64, select=sel)
    X1, e1, _ = _host_solve(zz, S, T, 64, select=sel, ldx=703)
    assert np.array_equal(X1, X0) and np.array_equal(e1, e0)
    # status +j detected after the overlapped solve; X is not written
    Sb = np.array([[0.5, 0.1, 0.2, 0.1], [0.0, 1.0, 0.3, 0.2], [0.0, 1.0, 1.0, 0.3], [0, 0, 0, 2.0]], order="F")
    with pytest.raises(zz.ZZError) as ei:
        _host_solve(zz, Sb, np.eye(4, order="F"), 32)
    assert ei.value.status == 2
    # entries near Omega/4: the deferred pre-scale test re-solves on the device copy (R6)
    S2, T2, _ = gen.config("C1", seed=6)
    Xr, er, _ = solve(zz, S2, T2, mb=32)
    X2, e2, info = _host_solve(zz, np.asfortranarray(np.ldexp(S2, 1021)), np.asfortranarray(np.ldexp(T2, 1021)), 32)
    assert info["prescaled"] == 1
    assert np.array_equal(X2, Xr)


# ---- back-transformation W = V X (xTGEVC HOWMNY='B', include/zz.h zz_tgevc_back) ----

def _back(zz, S, T, V, mb=0, select=None, ldw=None, ldv=None):
    zz.set_tile(mb)
    m = S.shape[0]
    n = oracle.count_columns(S, select)
    Sd, Td, Vd = to_dev(S), to_dev(T), to_dev(V, ldv)
    W = None
    if ldw is not None:
        W = torch.full((max(n, 1), ldw), np.nan, dtype=torch.float64, device="cuda").t()[:m, :n]
    W, e = zz.tgevc_back(Sd, Td, Vd, select=select, W=W, n_sel=n)
    torch.cuda.synchronize()
    return W.cpu().numpy(), e.cpu().numpy(), zz.last_info()


@pytest.mark.parametrize("name,seed,mb", [("C1", 0, 32), ("C1", 1, 64), ("C1", 5, 32), ("C2", 0, 128), ("C2", 1, 64)])
def test_back_parity(zz, name, seed, mb):
    S, T, _ = gen.config(name, seed=seed)
    V = gen.orthogonal(S.shape[0], seed=seed)
    W, e, info = _back(zz, S, T, V, mb=mb)
    ref = oracle.tgevc_back(S, T, V)
    lay = checks.column_layout(None, None, S)
    raw, ali = checks.parity(W, ref["W"], lay)
    assert np.isfinite(W).all() and info["ms_back"] > 0
    assert ali.max() <= TOL and raw.max() <= TOL, (ali.max(), raw.max())
    for col, j, sz in lay:       # LAPACK normalisation of the back-transformed columns
        w = np.abs(W[:, col]) if sz == 1 else np.abs(W[:, col]) + np.abs(W[:, col + 1])
        assert abs(w.max() - 1.0) <= 4 * 2.0 ** -53


def test_back_select_ldw_and_residual(zz):
    S, T, _ = gen.config("C2", seed=2, m=700, n2=105)
    m = S.shape[0]
    V = gen.orthogonal(m, seed=3)
    Q = gen.orthogonal(m, seed=4)
    W0, e0, _ = _back(zz, S, T, V, mb=64)
    W1, e1, _ = _back(zz, S, T, V, mb=64, ldw=703)        # odd ldw: bitwise the same
    assert np.array_equal(W0, W1) and np.array_equal(e0, e1)
    W2, e2, _ = _back(zz, S, T, V, mb=64, ldv=701)        # odd ldv (aligned copy of V)
    assert np.array_equal(W0, W2) and np.array_equal(e0, e2)
    sel = np.zeros(m, np.int32)
    sel[::7] = 1
    Ws, es, _ = _back(zz, S, T, V, mb=64, select=sel)
    lay_f = checks.column_layout(None, None, S)
    lay_s = checks.column_layout(None, None, S, sel)
    start = {j: col for col, j, _ in lay_f}
    for col, j, sz in lay_s:      # a selected column is the full solve's column, bit for bit
        assert np.array_equal(Ws[:, col:col + sz], W0[:, start[j]:start[j] + sz])
    # residual on the original pencil A = Q S V^T, B = Q T V^T
    ref = oracle.tgevc(S, T)
    D, Bm, _ = checks.build_DB(ref["pairs"], S)
    assert checks.residual(Q @ S @ V.T, Q @ T @ V.T, W0, D, Bm) <= 10 * m * 2.0 ** -53


# ---- left eigenvectors (xTGEVC SIDE='L', include/zz.h zz_tgevc_left) ----

def _left(zz, S, T, mb=0, select=None, ldy=None):
    zz.set_tile(mb)
    m = S.shape[0]
    n = oracle.count_columns(S, select)
    Y = None
    if ldy is not None:
        Y = torch.full((max(n, 1), ldy), np.nan, dtype=torch.float64, device="cuda").t()[:m, :n]
    Y, e = zz.tgevc_left(to_dev(S), to_dev(T), select=select, Y=Y, n_sel=n)
    torch.cuda.synchronize()
    return Y.cpu().numpy(), e.cpu().numpy(), zz.last_info()


@pytest.mark.parametrize("name,seed,mb", [("C1", 0, 32), ("C1", 3, 64), ("C2", 0, 128), ("C2", 2, 64)])
def test_left_parity(zz, name, seed, mb):
    S, T, _ = gen.config(name, seed=seed)
    Y, e, info = _left(zz, S, T, mb=mb)
    ref = oracle.tgevc_left(S, T)
    lay = checks.column_layout(None, None, S)
    raw, ali = checks.parity(Y, ref["Y"], lay)
    assert np.isfinite(Y).all() and (e <= 0).all()
    assert ali.max() <= TOL and raw.max() <= TOL, (ali.max(), raw.max())
    for col, j, sz in lay:
        assert np.all(Y[:j, col:col + sz] == 0.0)
        if sz == 2:
            assert e[col] == e[col + 1]


def test_left_select_ldy_and_errors(zz):
    S, T, _ = gen.config("C2", seed=1, m=700, n2=105)
    m = S.shape[0]
    Y0, e0, _ = _left(zz, S, T, mb=64)
    Y1, e1, _ = _left(zz, S, T, mb=64, ldy=701)
    assert np.array_equal(Y0, Y1) and np.array_equal(e0, e1)
    sel = np.zeros(m, np.int32)
    sel[3::11] = 1
    Ys, es, _ = _left(zz, S, T, mb=64, select=sel)
    lay_f = checks.column_layout(None, None, S)
    lay_s = checks.column_layout(None, None, S, sel)
    start = {j: col for col, j, _ in lay_f}
    for col, j, sz in lay_s:
        assert np.array_equal(Ys[:, col:col + sz], Y0[:, start[j]:start[j] + sz])
    # status codes refer to S: a 2x2 block with real eigenvalues at rows 2-3 (1-based) -> +2
    S2 = np.array([[0.5, 0.1, 0.2, 0.1], [0.0, 1.0, 0.3, 0.2], [0.0, 1.0, 1.0, 0.3], [0, 0, 0, 2.0]], order="F")
    with pytest.raises(zz.ZZError) as ei:
        _left(zz, S2, np.eye(4, order="F"), mb=32)
    assert ei.value.status == 2 == oracle.tgevc_left(S2, np.eye(4, order="F"))["status"]
    S3 = S2.copy()
    S3[3, 2] = 1.0
    with pytest.raises(zz.ZZError) as ei:
        _left(zz, S3, np.eye(4, order="F"), mb=32)
    assert ei.value.status == -105


def test_lower_parts_never_read(zz):
    # the contract the multi-GPU broadcast relies on (dist.broadcast_upper sends only the
    # upper trapezoid): NaN below the subdiagonal of S and below the diagonal of T changes
    # nothing, bit for bit
    S, T, _ = gen.config("C2", seed=0, m=600, n2=90)
    X0, e0, _ = solve(zz, S, T, mb=64)
    Sn, Tn = S.copy(order="F"), T.copy(order="F")
    il = np.tril_indices(600, -2)
    Sn[il] = np.nan
    Tn[np.tril_indices(600, -1)] = np.nan
    X1, e1, _ = solve(zz, Sn, Tn, mb=64)
    assert np.array_equal(X0, X1) and np.array_equal(e0, e1)


# ---- step grouping of the wavefront (zz_set_fusion 1 / 2 / 3) ----

@pytest.mark.parametrize("fusion", [1, 2, 3, 4, 6])
def test_fusion_modes_parity_select_and_repeat(zz, fusion):
    zz.set_fusion(fusion)
    try:
        S, T, _ = gen.config("C2", seed=0)
        X0, e0, info = solve(zz, S, T, mb=64)       # 32 tiles: groups with remainders
        if fusion > 1:
            assert info["fused_pairs"] >= 32 // fusion - 1
        check_against_oracle(S, T, X0, e0)
        X1, e1, _ = solve(zz, S, T, mb=64)
        assert np.array_equal(X0, X1) and np.array_equal(e0, e1)
        # a selection whose first active tile opens mid-group: bitwise the full solve's columns
        m = S.shape[0]
        for lo in (m - 330, m - 260, m - 200, m - 130, m - 70):
            sel = np.zeros(m, np.int32)
            sel[lo::37] = 1
            sel[5:60:9] = 1
            Xs, es, _ = solve(zz, S, T, mb=64, select=sel)
            lay_f = checks.column_layout(None, None, S)
            lay_s = checks.column_layout(None, None, S, sel)
            start = {j: col for col, j, _ in lay_f}
            for col, j, sz in lay_s:
                assert np.array_equal(Xs[:, col:col + sz], X0[:, start[j]:start[j] + sz]), (lo, j)
    finally:
        zz.set_fusion(4)


@pytest.mark.parametrize("fusion", [1, 3, 5])
def test_fusion_modes_stress(zz, fusion):
    # the scaling decisions of the grouped steps on a pencil whose unprotected substitution
    # overflows: finite, scaled, componentwise backward stable
    zz.set_fusion(fusion)
    try:
        S, T = _stress(2000, 1)
        X, e, info = solve(zz, S, T, mb=64)
        assert np.isfinite(X).all() and info["n_scaled"] > 0 and (e <= 0).all()
        ref = oracle.tgevc(S, T)
        lay = checks.column_layout(None, None, S)
        w = checks.comp_backward_error(S, T, X, ref["pairs"], lay, S.shape[0])
        assert w <= 10 * S.shape[0] * U, w
    finally:
        zz.set_fusion(4)



# ---- lookahead schedule (zz_set_lookahead) ----

def test_lookahead_bitwise_and_parity(zz):
    # m = 4096: the automatic mode turns it on; results are bitwise those of the plain
    # schedule (no scaling triggers) and within the parity tolerance of the oracle
    S, T, _ = gen.config("C3", seed=2, m=4096, n2=614)
    try:
        zz.set_lookahead(0)
        X0, e0, _ = solve(zz, S, T, mb=128)
        zz.set_lookahead(1)
        X1, e1, info = solve(zz, S, T, mb=128)
        assert info["lookahead_redo"] == 0
        assert np.array_equal(X0, X1) and np.array_equal(e0, e1)
        check_against_oracle(S, T, X1, e1)
        # host path with lookahead: bitwise the device path
        Xh, eh, _ = _host_solve(zz, S, T, 128)
        assert np.array_equal(Xh, X0) and np.array_equal(eh, e0)
    finally:
        zz.set_lookahead(1)


def test_lookahead_forced_on_stress_recomputes(zz):
    # forced on a pencil that scales: the bound-based first decisions would over-scale, the
    # call is recomputed without lookahead -- bitwise the plain schedule
    S, T = _stress(2000, 2)
    try:
        zz.set_lookahead(0)
        X0, e0, _ = solve(zz, S, T, mb=64)
        zz.set_lookahead(2)
        X1, e1, info = solve(zz, S, T, mb=64)
        assert np.array_equal(X0, X1) and np.array_equal(e0, e1)
        assert info["lookahead_redo"] == 1
        # the same with an odd ldx (X solved in the library's aligned workspace): the
        # recomputation must land in the caller's X, not in the workspace
        X2, e2, info3 = solve(zz, S, T, mb=64, ldx=2001)
        assert info3["lookahead_redo"] == 1
        assert np.array_equal(X0, X2) and np.array_equal(e0, e2)
        # a small well-scaled pencil forced on: no redo, bitwise
        S2, T2, _ = gen.config("C2", seed=1)
        zz.set_lookahead(0)
        Y0, f0, _ = solve(zz, S2, T2, mb=64)
        zz.set_lookahead(2)
        Y1, f1, info2 = solve(zz, S2, T2, mb=64)
        assert info2["lookahead_redo"] == 0 and np.array_equal(Y0, Y1) and np.array_equal(f0, f1)
    finally:
        zz.set_lookahead(1)


def _assemble_shards(zz, Sd, Td, m, n, P, select=None):
    """X assembled from the one-GPU emulation of every shard p of P (include/zz.h
    zz_set_shard): each call writes only shard p's columns into their global positions"""
    X = torch.full((n, m), float("nan"), dtype=torch.float64, device="cuda").t()
    E = torch.full((n,), 12345, dtype=torch.int32, device="cuda")
    written = np.zeros(n, bool)
    sub = torch.diagonal(Sd, -1).cpu().numpy()
    for p in range(P):
        zz.set_shard(p, P)
        zz.tgevc(Sd, Td, select=select, X=X, col_scale_exp=E, n_sel=n)
        torch.cuda.synchronize()
        cols = zz.shard_columns(sub, m, P, p, select=select)
        Xn = X.cpu().numpy()
        # exactly the shard's columns are new; the others keep what they had
        newly = ~np.isnan(Xn).all(axis=0) & ~written
        assert np.array_equal(np.flatnonzero(newly), cols), p
        written |= newly
    zz.set_shard(0, 1)
    return X.cpu().numpy(), E.cpu().numpy()


@pytest.mark.parametrize("P", [2, 3, 8])
def test_shard_emulation_assembles_bitwise(zz, P):
    """X is bitwise independent of the number of ranks;
    emulated on one GPU with zz_set_shard, through the library's own pack/unpack kernels."""
    S, T, _ = gen.config("C2", seed=2)
    m = S.shape[0]
    Sd, Td = to_dev(S), to_dev(T)
    zz.set_tile(128)
    sel = None if P != 3 else (np.random.default_rng(3).random(m) < 0.4).astype(np.int32)
    n = oracle.count_columns(S, sel)
    Xf, ef, _ = solve(zz, S, T, mb=128, select=sel)
    Xa, Ea = _assemble_shards(zz, Sd, Td, m, n, P, select=sel)
    assert np.array_equal(Xa, Xf) and np.array_equal(Ea, ef)
    assert zz.load().zz_set_shard(3, 2) == -1 and zz.load().zz_set_shard(0, 0) == -2


def test_nccl_one_rank_collective_path(zz):
    """The collective code path on one GPU through a one-rank NCCL communicator: panel
    broadcast in consumption order, the receiving ranks' copy of S and T (shards p != 0), the
    gather through NCCL send/recv and the unpack -- bitwise equal to the plain call."""
    cases = [(gen.config("C2", seed=1), 128, (1, 3)), (gen.config("C3", seed=2, m=4096, n2=614), 128, (2,))]
    uid = zz.get_unique_id()
    assert len(uid) == 128
    try:
        for (S, T, _), mb, Ps in cases:
            zz.init(0)
            m = S.shape[0]
            Sd, Td = to_dev(S), to_dev(T)
            X0, e0, _ = solve(zz, S, T, mb=mb)
            zz.init(0, 1, 0, zz.get_unique_id())
            zz.set_tile(mb)
            X1, e1 = zz.tgevc(Sd, Td)
            torch.cuda.synchronize()
            assert np.array_equal(X1.cpu().numpy(), X0) and np.array_equal(e1.cpu().numpy(), e0)
            for P in Ps:
                if P > 1:
                    Xa, Ea = _assemble_shards(zz, Sd, Td, m, m, P)
                    assert np.array_equal(Xa, X0) and np.array_equal(Ea, e0)
            # end to end with host buffers through the collective host path
            Xh = np.full((m, m), np.nan, order="F")
            eh = np.zeros(m, np.int32)
            zz.tgevc_host(S, T, X=Xh, col_scale_exp=eh)
            assert np.array_equal(Xh, X0) and np.array_equal(eh, e0)
    finally:
        zz.init(0)


def test_multirank_collective_mock():
    """The collective zz_tgevc / zz_tgevc_host with 2 and 3 ranks: one host thread per rank,
    all on this GPU, NCCL replaced by the in-process transport of tests/mock_nccl (NCCL itself
    refuses two ranks on one device).  This runs the library's multi-rank code paths proper
    -- the subdiagonal and panel broadcasts with non-root receivers, the cyclic ownership,
    the grouped send/recv gather of the packed upper parts, the unpack on rank 0 -- and X must
    equal the plain solve bit for bit (with a selection, the lookahead schedule, both tile
    sizes and the host-buffer variant)."""
    import os
    import subprocess
    import sys
    from tests import mock_nccl
    so = mock_nccl.build()
    env = dict(os.environ, ZZ_NCCL_LIB=so)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "mock_nccl", "run_ranks.py")], env=env,
                       capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "all ok" in r.stdout


def test_graph_replay_bitwise(zz):
    """CUDA-graph capture / replay of the wavefront (include/zz.h zz_set_graphs): replays,
    a recapture after new input pointers or a new selection, and the lookahead schedule give
    the bits of plain stream launches."""
    cases = [(gen.config("C2", seed=4), 128, None), (gen.config("C3", seed=2, m=4096, n2=614), 128, None),
             (gen.config("C1", seed=2), 32, None)]
    try:
        for (S, T, _), mb, _ in cases:
            zz.set_graphs(False)
            X0, e0, _ = solve(zz, S, T, mb=mb)
            zz.set_graphs(True)
            Sd, Td = to_dev(S), to_dev(T)
            for rep in range(3):      # capture, then replays on the same pointers
                X1, e1, _ = solve(zz, S, T, mb=mb, Sd=Sd, Td=Td)
                assert np.array_equal(X1, X0) and np.array_equal(e1, e0), rep
            X2, e2, _ = solve(zz, S, T, mb=mb)   # new input tensors: recaptured
            assert np.array_equal(X2, X0) and np.array_equal(e2, e0)
            sel = (np.random.default_rng(1).random(S.shape[0]) < 0.3).astype(np.int32)
            zz.set_graphs(False)
            Xs0, es0, _ = solve(zz, S, T, mb=mb, select=sel, Sd=Sd, Td=Td)
            zz.set_graphs(True)
            for rep in range(2):
                Xs1, es1, _ = solve(zz, S, T, mb=mb, select=sel, Sd=Sd, Td=Td)
                assert np.array_equal(Xs1, Xs0) and np.array_equal(es1, es0)
    finally:
        zz.set_graphs(True)


@pytest.mark.parametrize("name,mb,teams", [("C2", 128, (1, 3, 4, 6, 12)), ("C2", 64, (1, 2, 4, 8, 16)),
                                           ("C1", 32, (1, 2, 4, 16)), ("stress1000", 128, (1, 4, 12))])
def test_diag_team_bitwise(zz, name, mb, teams):
    """Teams of warps per diagonal-solve task (include/zz.h zz_set_diag_team): every team
    size gives the bits of one warp per task (the same instructions on the same operands per
    column), with and without a selection and on a stress pencil whose scalings trigger; and
    the automatic choice is in parity with the oracle."""
    if name == "stress1000":
        S, T = _stress(1000, 1)
    else:
        S, T, _ = gen.config(name, seed=5)
    sel = (np.random.default_rng(2).random(S.shape[0]) < 0.2).astype(np.int32)
    try:
        for select in (None, sel):
            zz.set_diag_team(1)
            X0, e0, info0 = solve(zz, S, T, mb=mb, select=select)
            for w in teams + (0, -1):
                zz.set_diag_team(w)
                X1, e1, _ = solve(zz, S, T, mb=mb, select=select)
                assert np.array_equal(X1, X0) and np.array_equal(e1, e0), (name, mb, w)
            if name != "stress1000":
                check_against_oracle(S, T, X0, e0, select=select, info=info0)
    finally:
        zz.set_diag_team(0)
