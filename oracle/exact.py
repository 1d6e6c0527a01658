"""Exact rational checker for DD/QD products -- TEST INFRASTRUCTURE ONLY.

Every finite double is an integer multiple of 2^-1074, so scaling by 2^SHIFT
(SHIFT >= 1074) turns each DD/QD component into a Python integer and the
dot products sum_k a_ik b_kj into exact big-integer arithmetic.  This is
the "exact higher-precision oracle" of BASELINE.json's north_star and
SURVEY.md s8c; it follows the integer approach of the reference's own
tests/oracles.py:13-37 (exact dyadic checks via float.as_integer_ratio),
extended from scalars to sampled matrix entries.

bound_ratio() returns, for each sampled (i, j),

    |c_ij - (AB)_ij| / (4 * l * u * (|A||B|)_ij)

so a value <= 1 means the componentwise north_star bound holds.
"""

from fractions import Fraction

import numpy as np

SHIFT = 1100


def _to_int(x):
    """Exact integer value of float64 x times 2^SHIFT."""
    if x == 0.0:
        return 0
    num, den = float(x).as_integer_ratio()
    k = den.bit_length() - 1
    return num << (SHIFT - k)


def bound_ratio(a, b, c, rows, cols, u_exp):
    """Max over the sampled (rows x cols) entries of err / (4 l u |A||B|).

    ``u_exp`` is the unit-roundoff exponent: 104 for DD, 209 for QD
    (north_star).  Returns (max_ratio, n_checked).
    """
    l = a.shape[1]
    arows = {i: [sum(_to_int(v) for v in a[i, k].tolist()) for k in range(l)] for i in rows}
    bcols = {j: [sum(_to_int(v) for v in b[k, j].tolist()) for k in range(l)] for j in cols}
    worst = Fraction(0)
    n = 0
    for i in rows:
        ai = arows[i]
        for j in cols:
            bj = bcols[j]
            dot = 0
            absdot = 0
            for x, y in zip(ai, bj):
                p = x * y
                dot += p
                absdot += abs(p)
            cij = sum(_to_int(v) for v in c[i, j].tolist()) << SHIFT
            err = abs(cij - dot)
            n += 1
            if err == 0:
                continue
            if absdot == 0:
                return float("inf"), n
            ratio = Fraction(err << u_exp, 4 * l * absdot)
            if ratio > worst:
                worst = ratio
    return float(worst), n


def sample_indices(m, n, count, seed=0):
    """Deterministic sample of row and column indices (includes the edges)."""
    rng = np.random.default_rng(seed)
    rows = sorted(set([0, m - 1] + rng.integers(0, m, size=max(0, count - 2)).tolist()))
    cols = sorted(set([0, n - 1] + rng.integers(0, n, size=max(0, count - 2)).tolist()))
    return rows, cols
