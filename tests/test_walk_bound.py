"""Host pin of the integer inequality that ends a candidate walk in the scoring kernel
(csrc/score_kernel.cu, nbr_pair / stop_key; DESIGN.md §7 "H5/H6").

Lists are sorted by key = |2 i_m - C|^2 (half cells, C = the coarse cell's centre).  For an atom
in fine cell a of that coarse cell, A = 2 a - C, delta^2 = |A|^2, and with rho^2 the largest
squared cell offset the walk still needs, the kernel ends the walk at the first entry with

    key > 4 rho^2   and   key - 4 rho^2 > delta^2   and
    (key - 4 rho^2 - delta^2)^2 > 4 * (4 rho^2) * delta^2            (all in integers)

which must be exactly  key > (2 rho + delta)^2  (real arithmetic), and must never fire for an
entry with |i_m - a|^2 <= rho^2 (triangle inequality |2 i_m - C| <= 2 |i_m - a| + |2 a - C|).
This test re-derives both facts by brute force over small grids; it shares no code with the
kernel (the expression is retyped from the comment above, the reference is the real-number
definition)."""
from fractions import Fraction
import itertools
import math

import numpy as np


def kernel_end(key: int, rho4: int, d2: int) -> bool:
    """The kernel's test, in exact integers (rho4 = 4 rho^2)."""
    if not key > rho4:
        return False
    t = key - rho4
    if not t > d2:
        return False
    u = t - d2
    return u * u > 4 * rho4 * d2


def beyond_real(key: int, rho2: int, d2: int) -> bool:
    """key > (2 rho + delta)^2 decided exactly: key - 4 rho^2 - delta^2 > 4 rho delta, the
    right side being sqrt(16 rho^2 delta^2) compared through exact rational squares."""
    lhs = key - 4 * rho2 - d2
    if lhs <= 0:
        return False
    return Fraction(lhs * lhs) > Fraction(16 * rho2 * d2)


def test_integer_test_equals_real_definition():
    rng = np.random.default_rng(7)
    for _ in range(20000):
        rho2 = int(rng.integers(0, 5000))
        d2 = int(rng.integers(0, 3 * 31 * 31 + 1))
        key = int(rng.integers(0, 40000))
        assert kernel_end(key, 4 * rho2, d2) == beyond_real(key, rho2, d2), (key, rho2, d2)
    # boundary: key exactly (2 rho + delta)^2 with integer rho, delta does not end the walk
    for rho, delta in itertools.product(range(0, 12), range(0, 12)):
        key = (2 * rho + delta) ** 2
        assert not kernel_end(key, 4 * rho * rho, delta * delta)
        assert kernel_end(key + 1, 4 * rho * rho, delta * delta)


def test_never_ends_before_a_needed_entry():
    """Every entry within rho of the atom passes (brute force over a coarse cell and a ball of
    entries, shifts 1..3), and the bound is tight: some entry just outside the reach of the
    worst-case bound of the same cell is cut."""
    for s in (1, 2, 3):
        n = 1 << s
        msk = n - 1
        base = 5 * n                      # the coarse cell [base, base + n)^3
        C = 2 * base + msk                # its centre in half cells, per axis
        span = range(base - 9, base + n + 9)
        ents = np.array(list(itertools.product(span, span, span)), dtype=np.int64)
        key = ((2 * ents - C) ** 2).sum(1)
        cut_any = False
        for a in itertools.product(range(base, base + n), repeat=3):
            a = np.array(a)
            A = 2 * (a & msk) - msk
            assert np.array_equal(A, 2 * a - C)
            d2 = int((A * A).sum())
            dd = ((ents - a) ** 2).sum(1)
            for rho2 in (0, 1, 7, 16, 30):
                end = np.array([kernel_end(int(k), 4 * rho2, d2) for k in key])
                assert not np.any(end & (dd <= rho2)), (s, a, rho2)
                # entries the worst-case bound (delta = msk sqrt 3) keeps but this one cuts
                worst = key <= (2 * math.sqrt(rho2) + msk * math.sqrt(3.0)) ** 2
                cut_any = cut_any or bool(np.any(end & worst))
        assert cut_any or s == 1
