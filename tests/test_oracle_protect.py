"""Pins of the oracle's ProtectDivision / ProtectUpdate against the
SPEC worked examples (tests/golden/protect_examples.txt) and exact-rational properties."""
import os
import random
from fractions import Fraction

import pytest

import oracle

OMEGA = 2.0 ** 1023
GOLD = os.path.join(os.path.dirname(__file__), "golden", "protect_examples.txt")


def _val(tok):
    if tok == "O":
        return OMEGA
    if tok == "O/2":
        return OMEGA / 2
    return float.fromhex(tok) if tok.startswith(("0x", "-0x")) else float(tok)


def _examples():
    out = []
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        f, *args, e = line.split()
        out.append((f, [_val(a) for a in args], int(e)))
    return out


@pytest.mark.parametrize("f,args,e", _examples())
def test_spec_examples(f, args, e):
    got = oracle.protect_division(*args) if f == "division" else oracle.protect_update(*args)
    assert got == e


def _rand_mag(rng):
    k = rng.random()
    if k < 0.05:
        return 0.0
    if k < 0.10:
        return OMEGA
    if k < 0.15:
        return OMEGA * (1 - rng.random() * 2 ** -40)
    if k < 0.20:
        return rng.random() * 2.0 ** -1022  # subnormal
    return rng.random() * 2.0 ** rng.randint(-1074, 1022)


def test_protect_update_contract_exact():
    rng = random.Random(1234)
    Om = Fraction(OMEGA)
    for _ in range(40000):
        y, t, x = (min(_rand_mag(rng), OMEGA) for _ in range(3))
        e = oracle.protect_update(y, t, x)
        assert e <= 0
        xi = Fraction(2) ** e
        total = Fraction(y) + Fraction(t) * Fraction(x)
        assert xi * total <= Om, (y, t, x, e)
        if e < 0:  # near-optimal: at most a factor 4 too small
            assert Fraction(2) ** (e + 2) * total > Om, (y, t, x, e)
        if total <= Om / 4:
            assert e == 0


def test_protect_division_contract_exact():
    rng = random.Random(99)
    Om = Fraction(OMEGA)
    for _ in range(40000):
        b = min(_rand_mag(rng), OMEGA)
        t = _rand_mag(rng)
        if t == 0.0:
            t = 2.0 ** -1074
        e = oracle.protect_division(b, t)
        assert e <= 0
        xi = Fraction(2) ** e
        assert xi * Fraction(b) <= Fraction(t) * Om, (b, t, e)
        if Fraction(b) <= Fraction(t) * Om or t >= 1:
            assert e == 0
        else:
            assert Fraction(2) ** (e + 2) * Fraction(b) > Fraction(t) * Om, (b, t, e)
