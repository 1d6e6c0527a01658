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


# ---------------------------------------------------------------------------
# Scalar (reference scalar.py:95-251): an immutable DD/QD number on the host
# ---------------------------------------------------------------------------

def _algebra(kind):
    from . import hostarith as h
    if kind is Kind.DD:
        return {"add": h.dd_add, "sub": h.dd_sub, "mul": h.dd_mul, "div": h.dd_div,
                "sqrt": h.dd_sqrt, "neg": h.dd_neg, "zero": h.DD_ZERO,
                "from_float": h.dd_from_float, "to_float": h.dd_to_float}
    if kind is Kind.QD:
        return {"add": h.qd_add, "sub": h.qd_sub, "mul": h.qd_mul, "div": h.qd_div,
                "sqrt": h.qd_sqrt, "neg": h.qd_neg, "zero": h.QD_ZERO,
                "from_float": h.qd_from_float, "to_float": h.qd_to_float}
    raise ValueError("arbitrary-precision scalars are out of scope for this build")


class Scalar:
    """A DD ``(hi, lo)`` or QD ``(x0, x1, x2, x3)`` value with its precision.
    Immutable; arithmetic through the operators or the ``scalar_*``
    functions gives the reference's bits (``hostarith``)."""

    __slots__ = ("prec", "payload")

    def __init__(self, prec, payload):
        object.__setattr__(self, "prec", prec)
        object.__setattr__(self, "payload", tuple(float(c) for c in payload))

    def __setattr__(self, name, value):
        raise AttributeError("Scalar is immutable")

    @staticmethod
    def zero(prec):
        return Scalar(prec, _algebra(prec.kind)["zero"])

    @staticmethod
    def from_float(v, prec):
        return Scalar(prec, _algebra(prec.kind)["from_float"](v))

    @staticmethod
    def from_int(k, prec):
        """The integer rounded once to the format (exact when it fits)."""
        from mpmath import libmp
        return Scalar._from_mpf(libmp.from_int(int(k)), prec)

    @staticmethod
    def from_str(s, prec):
        """A decimal literal at the format's precision plus guard bits,
        rounded once (reference scalar.py:129-133)."""
        from mpmath import libmp
        return Scalar._from_mpf(libmp.from_str(s, prec.bits + 64, libmp.round_nearest), prec)

    @staticmethod
    def _from_mpf(v, prec):
        from .matrix import _round_mpf
        _algebra(prec.kind)
        return Scalar(prec, _round_mpf(v, prec))

    def to_float(self):
        return _algebra(self.prec.kind)["to_float"](self.payload)

    def is_zero(self):
        return all(c == 0.0 for c in self.payload)

    def __eq__(self, other):
        if not isinstance(other, Scalar):
            return NotImplemented
        return self.prec == other.prec and self.payload == other.payload

    def __hash__(self):
        return hash((self.prec, self.payload))

    def __repr__(self):
        return f"Scalar({self.prec}, {self.payload!r})"

    def __add__(self, other):
        return scalar_add(self, other)

    def __sub__(self, other):
        return scalar_sub(self, other)

    def __mul__(self, other):
        return scalar_mul(self, other)

    def __truediv__(self, other):
        return scalar_div(self, other)

    def __neg__(self):
        return scalar_neg(self)


def _binary(op, x, y):
    if x.prec != y.prec:
        from .errors import PrecisionMismatchError
        raise PrecisionMismatchError(f"operand precisions differ: {x.prec} vs {y.prec}")
    return Scalar(x.prec, _algebra(x.prec.kind)[op](x.payload, y.payload))


def scalar_add(x, y):
    return _binary("add", x, y)


def scalar_sub(x, y):
    return _binary("sub", x, y)


def scalar_mul(x, y):
    return _binary("mul", x, y)


def scalar_div(x, y):
    return _binary("div", x, y)


def scalar_sqrt(x):
    return Scalar(x.prec, _algebra(x.prec.kind)["sqrt"](x.payload))


def scalar_neg(x):
    return Scalar(x.prec, _algebra(x.prec.kind)["neg"](x.payload))
