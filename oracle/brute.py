"""Pure-Python brute force for tiny inputs -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Written straight from the definitions, independent of cats_oracle.c, so the C oracle can be
pinned against it on small cases:
  - Eq. 3: t = min{t' : F(t') >= k}, scanned literally over the sorted sample
    values augmented with 0, F evaluated with exact rationals (fractions.Fraction).
  - Eq. 1/2/4/5 for d, m <= a few dozen, with Python floats.
"""
from __future__ import annotations

import math
from fractions import Fraction


def empirical_cdf(mags, t_prime) -> Fraction:
    """F(t') = #{a <= t'} / N as an exact fraction."""
    mags = list(mags)
    return Fraction(sum(1 for a in mags if a <= t_prime), len(mags))


def fit_threshold(values, k: float) -> float:
    """Eq. 3 literally: smallest candidate t' (0 or a sample magnitude) with F(t') >= k.

    F is compared against the exact rational value of the double k (reading G5)."""
    mags = [abs(float(v)) for v in values]
    kk = Fraction(k)
    for cand in [0.0] + sorted(mags):
        if empirical_cdf(mags, cand) >= kk:
            return cand
    raise AssertionError("unreachable: F(max) = 1 >= k")


def rank_exact(k: float, n: int) -> int:
    """r = ceil(k*N) in exact rational arithmetic on the binary value of k."""
    return math.ceil(Fraction(k) * n)


def silu(u: float) -> float:
    """Eq. 2: u / (1 + e^{-u})."""
    if u >= 0:
        return u / (1.0 + math.exp(-u))
    e = math.exp(u)
    return u * e / (1.0 + e)


def cats_mlp_tiny(x, Wg, Wu, Wd, t):
    """One token, neuron-major weights given as nested lists [m][d]; returns (y, keep)."""
    d = len(x)
    m = len(Wg)
    v = [silu(sum(x[i] * Wg[j][i] for i in range(d))) for j in range(m)]
    keep = [1 if abs(vj) >= t else 0 for vj in v]
    x1 = [(v[j] * sum(x[i] * Wu[j][i] for i in range(d))) if keep[j] else 0.0 for j in range(m)]
    y = [sum(x1[j] * Wd[j][c] for j in range(m) if keep[j]) for c in range(d)]
    return y, keep
