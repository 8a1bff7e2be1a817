"""Pins of the oracle's nominal flop count (BASELINE.json north_star
"the nominal update flop count ... defined in the oracle"): F(select) = sum over the
selected columns c of 2 r_c (r_c - 1), i.e. 4 flops (one FMA with S, one with T) for every
(row i, source row k) with i < k <= r_c, r_c the 1-based last row of the column's block
(a complex pair counts as two columns).  Pinned against (i) the closed form of an all-1x1
pencil, (ii) brute-force enumeration of the (column, i, k) triples on small pencils with
pairs and selections, (iii) SURVEY.md's printed C1-C3 values; and bench.py's own count (the
product side reports F without importing oracle/) must equal it exactly."""
import os
import sys

import numpy as np
import pytest

import gen
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _brute(S, select=None):
    """4 x #{(column c, i, k): 1 <= i < k <= r_c} by enumeration (no closed form)"""
    m = S.shape[0]
    sub = np.diagonal(S, -1)
    f, j = 0, 0
    while j < m:
        sz = 2 if (j + 1 < m and sub[j] != 0.0) else 1
        r = j + sz
        if select is None or select[j] or (sz == 2 and select[j + 1]):
            for _ in range(sz):
                cnt = 0
                for k in range(1, r + 1):
                    for i in range(1, k):
                        cnt += 1
                f += 4 * cnt
        j += sz
    return float(f)


@pytest.mark.parametrize("m", [1, 2, 3, 17, 200])
def test_flops_closed_form_all_real(m):
    S, _, _ = gen.generate(m, 0, 1.0 / m, seed=m)
    assert oracle.flops(S) == 2.0 * m * (m + 1) * (m - 1) / 3.0


@pytest.mark.parametrize("m,n2,seed", [(1, 0, 0), (2, 1, 1), (7, 2, 2), (40, 12, 3), (97, 30, 4)])
def test_flops_brute_force_with_pairs_and_select(m, n2, seed):
    S, _, _ = gen.generate(m, n2, 1.0 / m, seed=seed)
    assert oracle.flops(S) == _brute(S)
    rng = np.random.default_rng(seed)
    for frac in (0.0, 0.3, 1.0):
        sel = (rng.random(m) < frac).astype(np.int32)
        assert oracle.flops(S, sel) == _brute(S, sel)


@pytest.mark.parametrize("name,printed", [("C1", 5.8976e5), ("C2", 5.3333e9), ("C3", 6.6667e11)])
def test_flops_printed_values_and_bench_count(name, printed):
    S, _, _ = gen.config(name, seed=0)
    m = S.shape[0]
    f = oracle.flops(S)
    # SURVEY.md s.8(c) O10 prints the all-1x1 value 2 m (m+1)(m-1)/3 to 5 digits; a pair at
    # 0-based rows (j, j+1) raises its first column's r from j+1 to j+2, i.e. adds
    # 2(j+2)(j+1) - 2(j+1)j = 4(j+1) -- exact closed form with pairs
    assert abs(2.0 * m * (m + 1) * (m - 1) / 3.0 - printed) <= 1e-4 * printed
    sub = np.diagonal(S, -1)
    pairs = [j for j in range(m - 1) if sub[j] != 0.0]
    assert f == 2.0 * m * (m + 1) * (m - 1) / 3.0 + sum(4.0 * (j + 1) for j in pairs)
    blocks = bench.blocks_from_sub(np.diagonal(S, -1).copy(), m)
    assert bench.nominal_flops(blocks) == f
    rng = np.random.default_rng(1)
    sel = (rng.random(m) < 0.1).astype(np.int32)
    assert bench.nominal_flops(blocks, sel) == oracle.flops(S, sel)
