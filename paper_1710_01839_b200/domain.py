"""Host restatement of the EFT-domain test (``csrc/domain.cuh``).

The mirror kernels form each TwoProd error with one DFMA; the reference
forms it with Veltkamp's split and Dekker's product (``_kernels.pyx:19-29``).
The two agree whenever the operands are finite, no split overflows
(|x| < 2^995), no product overflows and the error is representable
(smallest nonzero exponents summing to >= -900) -- the range the reference's
own ``eft.two_prod`` guards (``eft.py:19-24``).  Outside it every GPU launch
runs the Dekker kernel instead, so results stay the reference's (e.g. the
NaN of an overflowed split, reported as ``RangeError``).

The device computes the same six words with one scan per product
(``csrc/domain.cu``); this numpy version serves tests and diagnostics.
"""

import numpy as np


def words(x):
    """(max biased exponent, 2047 - min biased exponent of a nonzero
    component or 0 if none, non-finite flag) over every component."""
    bits = np.ascontiguousarray(x, dtype=np.float64).view(np.uint64).ravel()
    if bits.size == 0:
        return 0, 0, 0
    e = ((bits >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.int64)
    nonzero = (bits & np.uint64(0x7FFFFFFFFFFFFFFF)) != 0
    mx = int(e.max())
    mn = int((2047 - e[nonzero]).max()) if nonzero.any() else 0
    return mx, mn, int((e == 0x7FF).any())


def unsafe_words(wa, wb, margin_lo=0, margin_hi=0):
    """domain.cuh domain_unsafe."""
    if wa[2] or wb[2]:
        return True
    max_a, max_b = wa[0] - 1023 + margin_hi, wb[0] - 1023 + margin_hi
    if max_a >= 995 or max_b >= 995 or max_a + max_b >= 1000:
        return True
    if wa[1] == 0 or wb[1] == 0:
        return False
    min_a = (2047 - wa[1]) - 1023 - margin_lo
    min_b = (2047 - wb[1]) - 1023 - margin_lo
    return min_a + min_b < -900


def unsafe(a, b, margin_lo=0, margin_hi=0):
    """True when the product a*b needs the Dekker kernels."""
    return unsafe_words(words(a), words(b), margin_lo, margin_hi)
