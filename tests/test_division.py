"""The division rewrite the kernels use is exact (CPU only).

Kernels divide by w_c with Markstein's correction (csrc/common.cuh DIV_RCP):
q0 = RN(a*y), r = RN(a - w_c*q0) (one fma), q = RN(q0 + r*y) (one fma),
y = RN(1/w_c).  This must equal IEEE RN(a/w_c) bit for bit whenever
2^-959 < |a| < 2^959 (the kernels fall back to a true division outside).
fma is emulated exactly with Fractions (float(Fraction) rounds correctly).
"""

import random
from fractions import Fraction

import pytest


def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def markstein(a, wc):
    y = 1.0 / wc
    q0 = a * y
    r = fma(-wc, q0, a)
    return fma(r, y, q0)


@pytest.mark.parametrize("wc", [8.0 / 3.0, 6.0, 26.0, 3.0, 7.0])
def test_markstein_equals_ieee_division(wc):
    rng = random.Random(1234)
    for i in range(4000):
        if i % 2:
            a = rng.uniform(-4.0, 4.0)
        else:
            a = rng.uniform(1.0, 2.0) * 2.0 ** rng.randint(-900, 900) * rng.choice((-1.0, 1.0))
        assert markstein(a, wc).hex() == (a / wc).hex(), (a, wc)


def test_power_of_two_reciprocal_is_exact():
    rng = random.Random(7)
    for _ in range(2000):
        a = rng.uniform(-10, 10)
        assert (a * 0.25).hex() == (a / 4.0).hex()
