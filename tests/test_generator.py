"""The shared input generator (gen/): determinism, thread-count independence, structure
and the planted spectrum of the BASELINE.json configs."""
import numpy as np
import pytest

import gen


def test_determinism_and_threads():
    a = gen.config("C2", seed=1, nthreads=1)
    b = gen.config("C2", seed=1, nthreads=4)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    c = gen.config("C2", seed=2)
    assert not np.array_equal(a[0], c[0])


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_structure_and_spectrum(name):
    S, T, lam = gen.config(name, seed=0)
    cfg = gen.CONFIGS[name]
    m = cfg["m"]
    assert np.all(np.tril(T, -1) == 0)
    assert np.all(np.tril(S, -2) == 0)
    sub = np.diag(S, -1)
    assert np.count_nonzero(sub) == cfg["n2"]
    nz = np.flatnonzero(sub)
    assert np.all(np.diff(nz) >= 2)  # no overlapping 2x2 blocks
    # planted separation (R16)
    if name == "C1":
        d = np.abs(lam[:, None] - lam[None, :]) + np.eye(m) * 1e9
        assert d.min() >= cfg["gap"]
    # off-diagonal variance ~ var_off
    iu = np.triu_indices(m, 2)
    vals = S[iu]
    assert abs(vals.var() / cfg["var_off"] - 1) < 0.1


def test_zero_inf_counts():
    S, T, lam = gen.generate(1000, 150, 1e-3, seed=3, n_zero=11, n_inf=13)
    d = np.diag(S).copy()
    t = np.diag(T).copy()
    sub = np.diag(S, -1)
    one = np.ones(1000, bool)
    one[np.flatnonzero(sub)] = False
    one[np.flatnonzero(sub) + 1] = False
    assert np.sum((d == 0) & one) == 11
    assert np.sum((t == 0) & one) == 13


def test_stress_tiles_scaled():
    c = dict(gen.CONFIGS["C5"])
    c.update(m=1024, n2=150)
    S, T, lam = gen.generate(seed=0, **c)
    big = np.abs(S) > 1e90
    ntile = 8
    nup = ntile * (ntile - 1) // 2
    tiles = {(i // 128, j // 128) for i, j in zip(*np.nonzero(big))}
    assert len(tiles) == round(0.05 * nup)
    assert all(I < J for I, J in tiles)
