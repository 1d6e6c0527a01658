"""CPU oracle for the DD/QD GEMM hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package, and only as the checker / the timed CPU
reference.  The product package ``paper_1710_01839_b200`` never imports it.

Contents
--------
* ``liboracle.so`` (``mpmm_oracle.c``): a plain-C restatement of the
  reference kernels (``/root/reference/pkg/src/mpmm/_kernels.pyx``), built
  with the reference's strict-IEEE flags.  Wrapped here as numpy functions
  with the reference's ``(rows, cols, comps)`` AoS layout.
* ``strassen``: a restatement of the reference's Strassen recursion
  (``multiply.py:267-338``) over the C kernels.
* ``ref_kernels()``: the reference's OWN Cython kernel module compiled from
  ``/root/reference`` into ``oracle/_ref`` (``make -C oracle ref``), used to
  pin the restatement and as the ``"reference"`` CPU baseline.
* ``exact``: exact rational (Python integer) checks of the componentwise
  bound ``|c - c_exact| <= 4 l u (|A||B|)``.

Parity is pinned: ``tests/test_oracle_golden.py`` checks this oracle against
golden vectors the reference produced (``tests/golden/``) and against
``oracle/_ref`` when it has been built.
"""

import ctypes
import importlib.machinery
import importlib.util
import os
import sysconfig
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_P = ctypes.POINTER(ctypes.c_double)
_I = ctypes.c_int64


def lib():
    """Load (building on first use if needed) the C restatement."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.run(["make", "-C", _HERE, "liboracle.so"], check=True,
                           stdout=subprocess.DEVNULL)
        L = ctypes.CDLL(path)
        for name in ("oracle_dd_simple_rows", "oracle_qd_simple_rows"):
            getattr(L, name).argtypes = [_P, _I, _P, _I, _P, _I, _I, _I, _I, _I]
            getattr(L, name).restype = None
        for name in ("oracle_dd_block_cells", "oracle_qd_block_cells"):
            getattr(L, name).argtypes = [_P, _I, _P, _I, _P, _I, _I, _I, _I, _I, _I, _I]
            getattr(L, name).restype = None
        for name in ("oracle_dd_ewise", "oracle_qd_ewise"):
            getattr(L, name).argtypes = [_P, _I, _P, _I, _P, _I, _I, _I, _I, ctypes.c_int]
            getattr(L, name).restype = None
        for name in ("oracle_two_prod", "oracle_two_sum"):
            getattr(L, name).argtypes = [ctypes.c_double, ctypes.c_double, _P]
        for name in ("oracle_dd_add", "oracle_dd_mul"):
            getattr(L, name).argtypes = [_P, _P, _P]
        L.oracle_qd_mul_add.argtypes = [_P, _P, _P]
        L.oracle_compress4.argtypes = [_P, ctypes.c_int, _P]
        _LIB = L
    return _LIB


def _ptr(x):
    assert x.dtype == np.float64 and x.flags.c_contiguous
    return x.ctypes.data_as(_P)


def _comps(x):
    return x.shape[2]


def _prefix(x):
    return "dd" if _comps(x) == 2 else "qd"


# ---------------------------------------------------------------------------
# the eight reference kernels, numpy signatures as in _kernels.pyx
# ---------------------------------------------------------------------------

def simple_rows(a, b, c, i0, i1):
    """_kernels.pyx:36-100 / :344-363 (dd/qd_simple_rows)."""
    fn = getattr(lib(), f"oracle_{_prefix(a)}_simple_rows")
    fn(_ptr(a), a.shape[1], _ptr(b), b.shape[1], _ptr(c), c.shape[1],
       a.shape[1], b.shape[1], i0, i1)


def block_cells(a, b, c, n_min, cell0, cell1):
    """_kernels.pyx:103-186 / :366-404 (dd/qd_block_cells); accumulates into c."""
    fn = getattr(lib(), f"oracle_{_prefix(a)}_block_cells")
    fn(_ptr(a), a.shape[1], _ptr(b), b.shape[1], _ptr(c), c.shape[1],
       a.shape[0], a.shape[1], b.shape[1], n_min, cell0, cell1)


def ewise(x, y, out, i0, i1, subtract):
    """_kernels.pyx:207-230 / :407-452 (dd/qd_ewise_add/sub)."""
    fn = getattr(lib(), f"oracle_{_prefix(x)}_ewise")
    fn(_ptr(x), x.shape[1], _ptr(y), y.shape[1], _ptr(out), out.shape[1],
       x.shape[1], i0, i1, 1 if subtract else 0)


# ---------------------------------------------------------------------------
# whole products (multiply.py:86-182 partitioning restated)
# ---------------------------------------------------------------------------

def _split_range(total, parts):
    """multiply.py:86-96."""
    parts = max(1, min(parts, total))
    base, rem = divmod(total, parts)
    out, lo = [], 0
    for p in range(parts):
        hi = lo + base + (1 if p < rem else 0)
        if hi > lo:
            out.append((lo, hi))
        lo = hi
    return out


def _run(worker, total, threads):
    """multiply.py:99-112 -- the C kernels release the GIL (ctypes does)."""
    if total == 0:
        return
    bounds = _split_range(total, threads)
    if threads == 1 or len(bounds) == 1:
        worker(0, total)
        return
    with ThreadPoolExecutor(max_workers=len(bounds)) as pool:
        for f in [pool.submit(worker, lo, hi) for lo, hi in bounds]:
            f.result()


def matmul_simple(a, b, threads=1, kernels=None):
    k = kernels
    c = np.zeros((a.shape[0], b.shape[1], _comps(a)))
    fn = (lambda lo, hi: simple_rows(a, b, c, lo, hi)) if k is None else \
        (lambda lo, hi: getattr(k, f"{_prefix(a)}_simple_rows")(a, b, c, lo, hi))
    _run(fn, a.shape[0], threads)
    return c


def matmul_block(a, b, n_min, threads=1, kernels=None, c=None):
    k = kernels
    if c is None:
        c = np.zeros((a.shape[0], b.shape[1], _comps(a)))
    cells = (-(-a.shape[0] // n_min)) * (-(-b.shape[1] // n_min))
    fn = (lambda lo, hi: block_cells(a, b, c, n_min, lo, hi)) if k is None else \
        (lambda lo, hi: getattr(k, f"{_prefix(a)}_block_cells")(a, b, c, n_min, lo, hi))
    _run(fn, cells, threads)
    return c


def ewise_new(x, y, subtract):
    out = np.zeros_like(x)
    ewise(x, y, out, 0, x.shape[0], subtract)
    return out


def _pad(x, size):
    if x.shape[0] == size and x.shape[1] == size:
        return x
    out = np.zeros((size, size, x.shape[2]))
    out[:x.shape[0], :x.shape[1]] = x
    return out


def strassen(a, b, cutoff, leaf_n_min):
    """multiply.py:293-338 _strassen_rec, serial; square inputs."""
    n = a.shape[0]
    if n <= cutoff:
        return matmul_block(a, b, leaf_n_min)
    even = n + (n & 1)
    ap, bp = _pad(a, even), _pad(b, even)
    h = even // 2
    q = lambda m, i, j: np.ascontiguousarray(m[i * h:(i + 1) * h, j * h:(j + 1) * h])
    a11, a12, a21, a22 = q(ap, 0, 0), q(ap, 0, 1), q(ap, 1, 0), q(ap, 1, 1)
    b11, b12, b21, b22 = q(bp, 0, 0), q(bp, 0, 1), q(bp, 1, 0), q(bp, 1, 1)
    E = ewise_new
    ops = (
        (E(a11, a22, False), E(b11, b22, False)),
        (E(a21, a22, False), b11),
        (a11, E(b12, b22, True)),
        (a22, E(b21, b11, True)),
        (E(a11, a12, False), b22),
        (E(a21, a11, True), E(b11, b12, False)),
        (E(a12, a22, True), E(b21, b22, False)),
    )
    p1, p2, p3, p4, p5, p6, p7 = (strassen(x, y, cutoff, leaf_n_min) for x, y in ops)
    c11 = E(E(E(p1, p4, False), p5, True), p7, False)
    c12 = E(p3, p5, False)
    c21 = E(p2, p4, False)
    c22 = E(E(E(p1, p3, False), p2, True), p6, False)
    c = np.zeros((even, even, a.shape[2]))
    c[:h, :h], c[:h, h:], c[h:, :h], c[h:, h:] = c11, c12, c21, c22
    return np.ascontiguousarray(c[:n, :n])


# ---------------------------------------------------------------------------
# scalar helpers (for DD/QD op known-answer tests)
# ---------------------------------------------------------------------------

def two_prod(a, b):
    out = (ctypes.c_double * 2)()
    lib().oracle_two_prod(a, b, out)
    return out[0], out[1]


def compress4(terms):
    t = np.ascontiguousarray(terms, dtype=np.float64)
    out = np.zeros(4)
    lib().oracle_compress4(_ptr(t), len(t), _ptr(out))
    return tuple(out)


# ---------------------------------------------------------------------------
# the reference's own compiled kernels (oracle/_ref)
# ---------------------------------------------------------------------------

def ref_kernels():
    """The reference's Cython kernel module built by ``make -C oracle ref``,
    or None when it has not been built."""
    path = os.path.join(_HERE, "_ref", "_kernels" + sysconfig.get_config_var("EXT_SUFFIX"))
    if not os.path.exists(path):
        return None
    loader = importlib.machinery.ExtensionFileLoader("_kernels", path)
    spec = importlib.util.spec_from_file_location("_kernels", path, loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    return mod


# ---------------------------------------------------------------------------
# the reference's slice predictor (predict.py:37-50), for the "CPU, predicted"
# baseline at sizes where a full reference run takes tens of minutes
# ---------------------------------------------------------------------------

DEFAULT_SLICE_MULTIPLIER = 2   # predict.py:20


def slice_rows_for(n_min, m, slice_multiplier=DEFAULT_SLICE_MULTIPLIER):
    """predict.py:37-42: rows of A in the timed slice, min(k * n_min, m)."""
    if n_min < 1 or m < 1 or slice_multiplier < 1:
        raise ValueError("block size, row count and multiplier must be positive")
    return min(slice_multiplier * n_min, m)


def predict_full_time(slice_time_s, m, n_min, slice_multiplier=DEFAULT_SLICE_MULTIPLIER):
    """predict.py:45-50: the slice time scaled by m / slice rows."""
    if slice_time_s <= 0.0:
        raise ValueError("slice time must be positive")
    return slice_time_s * (m / slice_rows_for(n_min, m, slice_multiplier))
