"""Precision tokens and their properties (the reference's ``PrecisionSpec``
and ``Kind``, ``scalar.py:26-89``).

The GPU path serves the two fixed families -- double-double (2 float64
components, 106 mantissa bits) and quad-double (4 components, 212 bits).
``ap:<bits>`` tokens still parse, so tables written by the reference load,
but every product entry point rejects them (arbitrary precision is outside
this build).
"""

import enum
from dataclasses import dataclass


class Kind(enum.Enum):
    DD = "dd"
    QD = "qd"
    AP = "ap"


# family -> (mantissa bits, float64 components, u of the north_star GEMM bound)
_FIXED = {Kind.DD: (106, 2, -104), Kind.QD: (212, 4, -209)}
AP_BITS_RANGE = (24, 1 << 20)
DD_BITS, QD_BITS = _FIXED[Kind.DD][0], _FIXED[Kind.QD][0]


@dataclass(frozen=True)
class PrecisionSpec:
    kind: Kind
    bits: int

    def __post_init__(self):
        if self.kind in _FIXED:
            want = _FIXED[self.kind][0]
            if self.bits != want:
                raise ValueError(f"{self.kind.value} carries a fixed {want}-bit mantissa")
        elif not AP_BITS_RANGE[0] <= self.bits <= AP_BITS_RANGE[1]:
            raise ValueError("big-float mantissa bits must lie in "
                             f"[{AP_BITS_RANGE[0]}, {AP_BITS_RANGE[1]}]")

    @classmethod
    def dd(cls):
        return cls(Kind.DD, DD_BITS)

    @classmethod
    def qd(cls):
        return cls(Kind.QD, QD_BITS)

    @classmethod
    def ap(cls, bits):
        return cls(Kind.AP, int(bits))

    @classmethod
    def parse(cls, token):
        """``dd``, ``qd`` or ``ap:<bits>``, case and surrounding space ignored."""
        tok = token.strip().lower()
        fixed = {k.value: k for k in _FIXED}
        if tok in fixed:
            return cls(fixed[tok], _FIXED[fixed[tok]][0])
        head, sep, tail = tok.partition(":")
        if head == "ap" and sep and tail.isdigit():
            return cls.ap(int(tail))
        raise ValueError(f"bad precision token {token!r}")

    @property
    def token(self):
        return f"ap:{self.bits}" if self.kind is Kind.AP else self.kind.value

    @property
    def comps(self):
        """float64 components per element (the trailing array dimension)."""
        if self.kind not in _FIXED:
            raise ValueError("arbitrary precision has no fixed component count")
        return _FIXED[self.kind][1]

    @property
    def unit_roundoff_exp(self):
        return -self.bits

    def unit_roundoff(self):
        """2^-bits, the reference's u (its verify bounds use it)."""
        return 2.0 ** -self.bits

    @property
    def gemm_bound_u(self):
        """The u of the north_star bound |c - c_exact| <= 4 l u (|A||B|):
        2^-104 (DD) or 2^-209 (QD)."""
        return 2.0 ** _FIXED[self.kind][2]

    def __str__(self):
        return self.token
