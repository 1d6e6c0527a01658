"""Dense DD/QD matrices on the host or in HBM (reference ``matrix.py``).

Layout contract (reference ``matrix.py:1-20,43-48``): a matrix of ``rows x
cols`` DD (QD) elements is ONE C-contiguous float64 array of shape
``(rows, cols, 2)`` (``(rows, cols, 4)``), array-of-structures.  The same
layout lives in HBM as a ``torch.float64`` CUDA tensor of the same shape,
so a host array crosses to the device with one contiguous copy and the
kernels read 16-byte ``{hi, lo}`` pairs (32-byte QD elements) with
vectorised loads; no re-layout ever happens.

``DenseMatrix.data`` is therefore either a ``numpy.ndarray`` (host) or a
``torch.Tensor`` on a CUDA device.  Products return their result where the
left operand lives.  Equality is bitwise (``np.array_equal`` semantics, as
the reference's ``__eq__``, matrix.py:91-98).
"""

from dataclasses import dataclass

import numpy as np

from .errors import PrecisionMismatchError, RangeError, ShapeError
from .scalar import Kind, PrecisionSpec


def _torch():
    import torch
    return torch


def _is_tensor(x):
    return type(x).__module__.startswith("torch") and hasattr(x, "data_ptr")


class DenseMatrix:
    __slots__ = ("rows", "cols", "prec", "data")

    def __init__(self, rows, cols, prec, data):
        if rows < 1 or cols < 1:
            raise ShapeError("matrix dimensions must be positive")
        if prec.kind is Kind.AP:
            raise ValueError("arbitrary precision (ap:<bits>) is out of scope for the GPU build")
        want = (rows, cols, prec.comps)
        if tuple(data.shape) != want:
            raise ShapeError(f"component array shape {tuple(data.shape)} != {want}")
        if _is_tensor(data):
            torch = _torch()
            if data.dtype != torch.float64 or not data.is_contiguous():
                raise TypeError("device data must be a contiguous float64 tensor")
        elif not (isinstance(data, np.ndarray) and data.dtype == np.float64):
            raise TypeError("host data must be a float64 numpy array")
        self.rows = rows
        self.cols = cols
        self.prec = prec
        self.data = data

    # -- construction -------------------------------------------------------

    @staticmethod
    def zeros(rows, cols, prec, device=None):
        """Zero matrix on the host (device=None) or on a CUDA device."""
        if device is None:
            return DenseMatrix(rows, cols, prec, np.zeros((rows, cols, prec.comps)))
        torch = _torch()
        return DenseMatrix(rows, cols, prec,
                           torch.zeros((rows, cols, prec.comps), dtype=torch.float64,
                                       device=device))

    @staticmethod
    def empty(rows, cols, prec, device):
        torch = _torch()
        return DenseMatrix(rows, cols, prec,
                           torch.empty((rows, cols, prec.comps), dtype=torch.float64,
                                       device=device))

    @staticmethod
    def from_ints(rows_of_ints, prec):
        """Exact integer matrix (reference matrix.py:64-67)."""
        m = len(rows_of_ints)
        n = len(rows_of_ints[0])
        out = DenseMatrix.zeros(m, n, prec)
        for i, row in enumerate(rows_of_ints):
            if len(row) != n:
                raise ShapeError("ragged rows")
            for j, v in enumerate(row):
                out.data[i, j] = _int_components(int(v), prec.comps)
        return out

    @staticmethod
    def identity(n, prec):
        out = DenseMatrix.zeros(n, n, prec)
        for i in range(n):
            out.data[i, i, 0] = 1.0
        return out

    # -- residency ----------------------------------------------------------

    @property
    def is_device(self):
        return _is_tensor(self.data)

    @property
    def device(self):
        return self.data.device if self.is_device else None

    def to_device(self, device=None):
        """This matrix in HBM (no copy when it already is)."""
        if self.is_device:
            return self
        torch = _torch()
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        host = torch.from_numpy(np.ascontiguousarray(self.data))
        return DenseMatrix(self.rows, self.cols, self.prec, host.to(dev, non_blocking=False))

    def to_host(self):
        """Host copy through a pinned (page-locked) buffer, so the D2H runs
        at full PCIe/C2C bandwidth; the numpy array owns the buffer."""
        if not self.is_device:
            return self
        torch = _torch()
        out = torch.empty(tuple(self.data.shape), dtype=torch.float64, pin_memory=True)
        out.copy_(self.data)
        return DenseMatrix(self.rows, self.cols, self.prec, out.numpy())

    def host_array(self):
        return self.to_host().data

    # -- element access ------------------------------------------------------

    def get(self, i, j):
        """Element (i, j) as a Scalar (reference matrix.py:79-83); its
        ``payload`` is the tuple of float components."""
        from .scalar import Scalar
        if self.is_device:
            return Scalar(self.prec, self.data[i, j].cpu().tolist())
        return Scalar(self.prec, self.data[i, j].tolist())

    def to_float_array(self):
        """Lossy double view (reference matrix.py:85-89)."""
        return self.host_array().sum(axis=2)

    def __eq__(self, other):
        if not isinstance(other, DenseMatrix):
            return NotImplemented
        if (self.rows, self.cols, self.prec) != (other.rows, other.cols, other.prec):
            return False
        return bool(np.array_equal(self.host_array(), other.host_array()))

    __hash__ = None

    def __repr__(self):
        where = "cuda" if self.is_device else "host"
        return f"DenseMatrix({self.rows}x{self.cols}, {self.prec}, {where})"


def _int_components(v, comps):
    out = []
    rest = v
    for _ in range(comps):
        c = float(rest)
        out.append(c)
        rest -= int(c)
    return tuple(out)


def leading_rows(mat, r):
    """The first ``r`` rows, sharing storage (reference matrix.py:111-117)."""
    if not 1 <= r <= mat.rows:
        raise ShapeError(f"cannot take {r} leading rows of {mat.rows}")
    return DenseMatrix(r, mat.cols, mat.prec, mat.data[:r])


# ---------------------------------------------------------------------------
# block partitions (reference matrix.py:124-161)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class BlockPartition:
    n_min: int
    row_extents: tuple
    inner_extents: tuple
    col_extents: tuple

    @property
    def m_blocks(self):
        return len(self.row_extents)

    @property
    def l_blocks(self):
        return len(self.inner_extents)

    @property
    def n_blocks(self):
        return len(self.col_extents)


def _extents(dim, n_min):
    full, rem = divmod(dim, n_min)
    return (n_min,) * full + ((rem,) if rem else ())


def make_partition(m, l, n, n_min):
    """Ceil-divide each axis into blocks of at most ``n_min``."""
    if n_min < 1:
        raise ShapeError("block size must be positive")
    return BlockPartition(n_min, _extents(m, n_min), _extents(l, n_min), _extents(n, n_min))


# ---------------------------------------------------------------------------
# the paper's test pair (reference matrix.py:168-200)
# ---------------------------------------------------------------------------

_GUARD_BITS = 64


def _components_from_mpf(x, count):
    from mpmath import libmp
    comps, rest = [], x
    for _ in range(count):
        c = libmp.to_float(rest, rnd=libmp.round_nearest)
        comps.append(c)
        rest = libmp.mpf_sub(rest, libmp.from_float(c), 0, libmp.round_nearest)
    return comps


def _round_mpf(x, prec):
    """Round a wide big-float into DD (quick-two-sum normalised) or QD
    (renormalised) components, as the reference's Scalar._from_ap_exactish
    (scalar.py:141-149)."""
    c = _components_from_mpf(x, prec.comps)
    if prec.kind is Kind.DD:
        s = c[0] + c[1]
        return (s, c[1] - (s - c[0]))
    from .inputs import _renorm5_vec
    r = _renorm5_vec(*[np.array(v) for v in (c[0], c[1], c[2], c[3], 0.0)])
    return tuple(float(v) for v in r)


def generate_test_pair(n, prec):
    """A[i][j] = sqrt(5)(i+j-1), B[i][j] = sqrt(3)(n-i), 1-based indices
    (reference matrix.py:168-200).  Host matrices."""
    if n < 1:
        raise ShapeError("matrix dimension must be positive")
    from mpmath import libmp
    rnd = libmp.round_nearest
    guard = prec.bits + _GUARD_BITS
    sqrt5 = libmp.mpf_sqrt(libmp.from_int(5), guard, rnd)
    sqrt3 = libmp.mpf_sqrt(libmp.from_int(3), guard, rnd)
    a_vals = np.zeros((2 * n, prec.comps))
    for k in range(1, 2 * n):
        a_vals[k] = _round_mpf(libmp.mpf_mul(sqrt5, libmp.from_int(k), guard, rnd), prec)
    b_vals = np.zeros((n, prec.comps))
    for k in range(1, n):
        b_vals[k] = _round_mpf(libmp.mpf_mul(sqrt3, libmp.from_int(k), guard, rnd), prec)
    idx = np.arange(n)
    a = np.ascontiguousarray(a_vals[idx[:, None] + idx[None, :] + 1])
    b = np.ascontiguousarray(np.broadcast_to(b_vals[n - 1 - idx][:, None, :],
                                             (n, n, prec.comps)))
    return DenseMatrix(n, n, prec, a), DenseMatrix(n, n, prec, b)


# ---------------------------------------------------------------------------
# norms and comparison (reference matrix.py:207-294)
# ---------------------------------------------------------------------------

def frobenius_norm(mat):
    """Frobenius norm in working precision, as a double."""
    from . import _cuda
    rc, v = _cuda.host_frobenius_norm(mat.prec.comps, mat.host_array())
    _raise_norm(rc)
    return v


def frobenius_rel_diff(x, y):
    """``||X - Y||_F / ||Y||_F`` in working precision, as a double
    (``||X - Y||_F`` when ``||Y||_F`` is zero), evaluated with the
    reference's sequential DD/QD operation order."""
    if (x.rows, x.cols) != (y.rows, y.cols):
        raise ShapeError(f"shape mismatch: {x.rows}x{x.cols} vs {y.rows}x{y.cols}")
    if x.prec != y.prec:
        raise PrecisionMismatchError(f"precision mismatch: {x.prec} vs {y.prec}")
    from . import _cuda
    rc, v = _cuda.host_frobenius_rel_diff(x.prec.comps, x.host_array(), y.host_array())
    _raise_norm(rc)
    return v


def _raise_norm(rc):
    if rc == 1:
        raise RangeError("norm accumulation overflowed the working precision")
    if rc == 2:
        raise ValueError("square root of a negative value")
    if rc != 0:
        raise RuntimeError(f"norm helper failed with code {rc}")


__all__ = ["DenseMatrix", "BlockPartition", "make_partition", "leading_rows",
           "generate_test_pair", "frobenius_norm", "frobenius_rel_diff", "PrecisionSpec"]


# ---------------------------------------------------------------------------
# text dumps (the reference's write_matrix / read_matrix format)
# ---------------------------------------------------------------------------

def write_matrix(mat, fp):
    """One header line ``rows cols precision``, then a line per row: the
    elements separated by spaces, each element's components as hex floats
    joined by commas -- exact, and readable by the reference's
    read_matrix.  Device matrices are copied to the host first."""
    data = mat.host_array()
    fp.write(f"{mat.rows} {mat.cols} {mat.prec.token}\n")
    for row in data:
        fp.write(" ".join(",".join(float(c).hex() for c in el) for el in row) + "\n")


def read_matrix(fp):
    """Inverse of write_matrix (DD and QD dumps); a malformed dump raises
    TableFormatError."""
    from .errors import TableFormatError
    head = fp.readline().split()
    try:
        rows, cols, prec = int(head[0]), int(head[1]), PrecisionSpec.parse(head[2])
        comps = prec.comps
    except (IndexError, ValueError) as ex:
        raise TableFormatError(f"bad matrix dump header: {ex}") from None
    if len(head) != 3:
        raise TableFormatError("bad matrix dump header")
    data = np.zeros((rows, cols, comps))
    for i in range(rows):
        elems = fp.readline().split()
        if len(elems) != cols:
            raise TableFormatError(f"row {i} has {len(elems)} elements, expected {cols}")
        for j, el in enumerate(elems):
            parts = el.split(",")
            if len(parts) != comps:
                raise TableFormatError(f"element {i},{j} has {len(parts)} components")
            try:
                data[i, j] = [float.fromhex(p) for p in parts]
            except ValueError:
                raise TableFormatError(f"element {i},{j}: bad hex float") from None
    return DenseMatrix(rows, cols, prec, data)
