"""Precision descriptors (reference ``pkg/src/mpmm/scalar.py:26-89``).

Only the DD and QD families are on the GPU hot path.  ``ap:<bits>`` tokens
parse (so tables written by the reference load) but every product entry
point rejects them: arbitrary precision is out of scope.
"""

import enum
from dataclasses import dataclass

DD_BITS = 106
QD_BITS = 212
AP_MIN_BITS = 24
AP_MAX_BITS = 1 << 20


class Kind(enum.Enum):
    DD = "dd"
    QD = "qd"
    AP = "ap"


@dataclass(frozen=True)
class PrecisionSpec:
    kind: Kind
    bits: int

    def __post_init__(self):
        if self.kind is Kind.DD and self.bits != DD_BITS:
            raise ValueError("double-double carries a fixed 106-bit mantissa")
        if self.kind is Kind.QD and self.bits != QD_BITS:
            raise ValueError("quad-double carries a fixed 212-bit mantissa")
        if self.kind is Kind.AP and not (AP_MIN_BITS <= self.bits <= AP_MAX_BITS):
            raise ValueError(f"big-float mantissa bits must lie in [{AP_MIN_BITS}, {AP_MAX_BITS}]")

    @staticmethod
    def dd():
        return PrecisionSpec(Kind.DD, DD_BITS)

    @staticmethod
    def qd():
        return PrecisionSpec(Kind.QD, QD_BITS)

    @staticmethod
    def ap(bits):
        return PrecisionSpec(Kind.AP, int(bits))

    @staticmethod
    def parse(token):
        """Parse ``dd``, ``qd`` or ``ap:<bits>`` (scalar.py:60-74)."""
        token = token.strip().lower()
        if token == "dd":
            return PrecisionSpec.dd()
        if token == "qd":
            return PrecisionSpec.qd()
        if token.startswith("ap:"):
            try:
                bits = int(token[3:])
            except ValueError:
                raise ValueError(f"bad precision token {token!r}") from None
            return PrecisionSpec.ap(bits)
        raise ValueError(f"bad precision token {token!r}")

    @property
    def token(self):
        if self.kind is Kind.AP:
            return f"ap:{self.bits}"
        return self.kind.value

    @property
    def comps(self):
        """float64 components per element: 2 (DD) or 4 (QD)."""
        if self.kind is Kind.DD:
            return 2
        if self.kind is Kind.QD:
            return 4
        raise ValueError("arbitrary precision has no fixed component count")

    @property
    def unit_roundoff_exp(self):
        return -self.bits

    def unit_roundoff(self):
        """2^-bits, as in the reference (scalar.py:84-86).  Note that the
        north_star GEMM bound uses u = 2^-104 (DD) / 2^-209 (QD) instead;
        see ``gemm_bound_u``."""
        return 2.0 ** -self.bits

    @property
    def gemm_bound_u(self):
        """The u of the north_star componentwise bound 4 l u (|A||B|)."""
        return 2.0 ** -104 if self.kind is Kind.DD else 2.0 ** -209

    def __str__(self):
        return self.token
