"""Simple, blocked and Strassen products on the GPU (reference ``multiply.py``).

Public entry points keep the reference's names, arguments, validation and
exceptions (``multiply.py:25-79,115-182,267-350``) so existing callers work
unchanged; results are bit-identical to the reference CPU kernels:

* ``matmul_simple`` -- the triple loop, k ascending (one thread per element);
* ``matmul_block``  -- the blocked product; the block size ``n_min`` selects
  the CTA tile (a performance knob: results never depend on it, exactly as
  the reference's blocked == simple guarantee, multiply.py:171-176);
* ``matmul_strassen`` -- Eq. (3) recursion with the reference's padding,
  operand order and combination order, leaves on the blocked kernel,
  operand sums and quadrant combinations as fused elementwise kernels over
  strided quadrant views (no quadrant copies).

``threads`` is accepted and validated for signature compatibility; on the
GPU the parallelism is the CTA grid (and, across GPUs, ``shard.py``).
Inputs may live on the host (numpy) or in HBM (torch CUDA tensors); the
result lives where ``a`` lives.
"""

import enum
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _cuda, backend
from .errors import PrecisionMismatchError, RangeError, ShapeError
from .matrix import DenseMatrix
from .scalar import Kind


class Algorithm(enum.Enum):
    SIMPLE = "simple"
    BLOCK = "block"
    STRASSEN = "strassen"
    EXACT = "exact"     # extension: the int8 tensor-core exact mode (tensor.py)


DEFAULT_STRASSEN_CUTOFF = 64
DEFAULT_BLOCK_SIZE = 64


@dataclass(frozen=True)
class AlgorithmChoice:
    """One tuner outcome; tokens ``simple``, ``block:N``, ``strassen:C/N``
    (reference multiply.py:35-71), and ``exact`` for the opt-in exact
    tensor-core mode (``TuningConfig.exact``).  ``exact`` may carry the
    mirror block size to fall back to (``exact/N``) when an operand's
    dynamic range is too wide for the int8 CRT scheme."""
    kind: Algorithm
    n_min: Optional[int] = None
    cutoff: Optional[int] = None

    def __post_init__(self):
        if self.kind is Algorithm.BLOCK and (not self.n_min or self.n_min < 1):
            raise ValueError("blocked algorithm needs a positive block size")
        if self.kind is Algorithm.STRASSEN:
            if not self.cutoff or self.cutoff < 2:
                raise ValueError("Strassen needs a recursion cutoff >= 2")
            if not self.n_min or self.n_min < 1:
                raise ValueError("Strassen needs a positive leaf block size")

    @property
    def token(self):
        if self.kind is Algorithm.SIMPLE:
            return "simple"
        if self.kind is Algorithm.BLOCK:
            return f"block:{self.n_min}"
        if self.kind is Algorithm.EXACT:
            return "exact" if self.n_min is None else f"exact/{self.n_min}"
        return f"strassen:{self.cutoff}/{self.n_min}"

    @staticmethod
    def parse(tok):
        if tok == "simple":
            return AlgorithmChoice(Algorithm.SIMPLE)
        if tok.startswith("block:"):
            return AlgorithmChoice(Algorithm.BLOCK, n_min=int(tok[len("block:"):]))
        if tok.startswith("strassen:"):
            cut, _, leaf = tok[len("strassen:"):].partition("/")
            return AlgorithmChoice(Algorithm.STRASSEN, n_min=int(leaf), cutoff=int(cut))
        if tok == "exact":
            return AlgorithmChoice(Algorithm.EXACT)
        if tok.startswith("exact/"):
            return AlgorithmChoice(Algorithm.EXACT, n_min=int(tok[len("exact/"):]))
        raise ValueError(f"bad algorithm token {tok!r}")

    def __str__(self):
        return self.token


class StrassenStats:
    """Multiplication / addition counts of a Strassen run (multiply.py:74-79)."""

    def __init__(self):
        self.multiplications = 0
        self.additions = 0


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------

def _torch():
    import torch
    return torch


def _stream():
    return _torch().cuda.current_stream().cuda_stream


class _View:
    """A rows x cols window of a contiguous (R, C, comps) device tensor."""

    __slots__ = ("base", "r0", "c0", "rows", "cols")

    def __init__(self, base, r0, c0, rows, cols):
        self.base, self.r0, self.c0, self.rows, self.cols = base, r0, c0, rows, cols

    @staticmethod
    def of(t):
        return _View(t, 0, 0, t.shape[0], t.shape[1])

    @property
    def comps(self):
        return self.base.shape[2]

    @property
    def ld(self):
        return self.base.shape[1]

    @property
    def ptr(self):
        return self.base.data_ptr() + 8 * self.comps * (self.r0 * self.ld + self.c0)

    def sub(self, r0, c0, rows, cols):
        return _View(self.base, self.r0 + r0, self.c0 + c0, rows, cols)


def _gemm_view(algo, n_min, A, B, C, accumulate, flag=None):
    _cuda.gemm_dev(A.comps, algo, n_min, A.rows, A.cols, B.cols, A.ptr, A.ld, B.ptr, B.ld,
                   C.ptr, C.ld, accumulate, flag, _stream())


def _ewise_view(O, X, Y, sy, Z=None, sz=1, W=None, sw=1):
    _cuda.ewise_dev(X.comps, X.rows, X.cols, O.ptr, O.ld, X.ptr, X.ld, Y.ptr, Y.ld, sy,
                    Z.ptr if Z is not None else None, Z.ld if Z is not None else 0, sz,
                    W.ptr if W is not None else None, W.ld if W is not None else 0, sw,
                    _stream())


# ---------------------------------------------------------------------------
# validation (multiply.py:115-127)
# ---------------------------------------------------------------------------

def _check_pair(a, b, threads):
    if a.cols != b.rows:
        raise ShapeError(f"inner dimensions differ: {a.rows}x{a.cols} times {b.rows}x{b.cols}")
    if a.prec != b.prec:
        raise PrecisionMismatchError(f"operand precisions differ: {a.prec} vs {b.prec}")
    if threads < 1:
        raise ValueError("thread count must be positive")
    if a.prec.kind is Kind.AP:
        raise ValueError("arbitrary precision is out of scope for the GPU build")


def _check_finite(c, flag=None):
    if c.is_device:
        if flag is None:
            torch = _torch()
            flag = torch.zeros(1, dtype=torch.int32, device=c.data.device)
            _cuda.nonfinite_dev(c.prec.comps, c.rows, c.cols, c.data.data_ptr(), c.cols,
                                flag.data_ptr(), _stream())
        bad = bool(flag.item())
    else:
        bad = not np.isfinite(c.data).all()
    if bad:
        raise RangeError("matrix product overflowed the working precision")
    return c


def _flag(device):
    torch = _torch()
    return torch.zeros(1, dtype=torch.int32, device=device)


def _operands(a, b):
    """Device copies of the operands and whether the result goes home."""
    if backend.is_cuda():
        return a.to_device(), b.to_device(a.device), not a.is_device
    return a.to_host(), b.to_host(), False


def _result(c, to_host):
    return c.to_host() if to_host else c


def _pinned_empty(rows, cols, comps):
    torch = _torch()
    return torch.empty((rows, cols, comps), dtype=torch.float64, pin_memory=True).numpy()


def _host_product(a, b, algo, n_min):
    """Host operands, host result, one pipelined C-ABI call
    (mpmm_gemm_host: k-panel H2D overlapped with the GEMM, page-locked
    result buffer, finite flag from the GEMM epilogue)."""
    out = _pinned_empty(a.rows, b.cols, a.prec.comps)
    ok = _cuda.gemm_host(a.prec.comps, algo, n_min, np.ascontiguousarray(a.data),
                         np.ascontiguousarray(b.data), out, accumulate=False)
    if not ok:
        raise RangeError("matrix product overflowed the working precision")
    return DenseMatrix(a.rows, b.cols, a.prec, out)


# ---------------------------------------------------------------------------
# simple and blocked products (multiply.py:134-182)
# ---------------------------------------------------------------------------

def _split_range(total, parts):
    """multiply.py:86-96 (used for the host-protocol path)."""
    parts = max(1, min(parts, total))
    base, rem = divmod(total, parts)
    bounds, lo = [], 0
    for p in range(parts):
        hi = lo + base + (1 if p < rem else 0)
        if hi > lo:
            bounds.append((lo, hi))
        lo = hi
    return bounds


def _host_partitioned(worker, total, threads):
    if total == 0:
        return
    bounds = _split_range(total, threads)
    if len(bounds) == 1:
        worker(0, total)
        return
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(bounds)) as pool:
        for f in [pool.submit(worker, lo, hi) for lo, hi in bounds]:
            f.result()


def _simple_into(a, b, c, threads=1, flag=None):
    """c = a*b, simple algorithm, c overwritten (multiply.py:134-145)."""
    if c.is_device:
        _gemm_view(_cuda.ALGO_SIMPLE, 0, _View.of(a.data), _View.of(b.data), _View.of(c.data),
                   False, flag.data_ptr() if flag is not None else None)
        return
    kern = backend.kernels()
    fn = kern.dd_simple_rows if a.prec.kind is Kind.DD else kern.qd_simple_rows
    _host_partitioned(lambda lo, hi: fn(a.data, b.data, c.data, lo, hi), a.rows, threads)


def _block_into(a, b, c, n_min, threads=1, flag=None):
    """c += a*b over every cell of the n_min grid (multiply.py:148-160);
    the caller passes a zero c for a plain product."""
    cells = (-(-a.rows // n_min)) * (-(-b.cols // n_min))
    if c.is_device:
        _gemm_view(_cuda.ALGO_BLOCK, n_min, _View.of(a.data), _View.of(b.data),
                   _View.of(c.data), True, flag.data_ptr() if flag is not None else None)
        return
    kern = backend.kernels()
    fn = kern.dd_block_cells if a.prec.kind is Kind.DD else kern.qd_block_cells
    _host_partitioned(lambda lo, hi: fn(a.data, b.data, c.data, n_min, lo, hi), cells, threads)


# ---------------------------------------------------------------------------
# gpus= : several GPUs of this node from one process
# ---------------------------------------------------------------------------

def _gpu_list(gpus):
    """``gpus``: a count G (devices 0..G-1) or an explicit device list."""
    if isinstance(gpus, (int, np.integer)):
        if gpus < 1:
            raise ValueError("gpu count must be positive")
        return list(range(int(gpus)))
    devs = [int(g) for g in gpus]
    if not devs or min(devs) < 0:
        raise ValueError("gpu list must name devices")
    return devs


_runtime_devs = None


def _runtime(devs):
    """The native multi-GPU runtime (csrc/runtime.cpp: one NCCL communicator
    per device, ncclCommInitAll) over exactly ``devs``."""
    global _runtime_devs
    if _runtime_devs == devs:
        return
    if len(set(devs)) != len(devs):
        raise ValueError("row-sharded products need distinct devices")
    if _runtime_devs is not None:
        _cuda.runtime_finalize()
        _runtime_devs = None
    _cuda.runtime_init(len(devs), devs)
    _runtime_devs = list(devs)


def _rows_multi(a, b, algo, n_min, devs):
    """C's rows split over ``devs`` (64-row aligned blocks, mpmm_multi_plan),
    each GPU receiving its rows of A, B broadcast by NCCL in k-panels
    overlapped with the per-panel GEMMs; bitwise the one-GPU product (each
    element keeps one owner and its ascending k order)."""
    _runtime(devs)
    ha = np.ascontiguousarray(a.host_array())
    hb = np.ascontiguousarray(b.host_array())
    out = _pinned_empty(a.rows, b.cols, a.prec.comps)
    bad, _ = _cuda.gemm_multi(a.prec.comps, algo, n_min, 0, ha, hb, out)
    if bad:
        raise RangeError("matrix product overflowed the working precision")
    c = DenseMatrix(a.rows, b.cols, a.prec, out)
    return c.to_device(a.device) if a.is_device else c


def matmul_simple(a, b, threads=1, *, gpus=1):
    """Triple-loop product; k accumulated in ascending order.  ``gpus`` > 1
    row-shards C over that many GPUs of this node (bitwise the same C)."""
    _check_pair(a, b, threads)
    devs = _gpu_list(gpus)
    if len(devs) > 1:
        return _rows_multi(a, b, _cuda.ALGO_SIMPLE, 0, devs)
    if backend.is_cuda() and not a.is_device and not b.is_device:

        return _host_product(a, b, _cuda.ALGO_SIMPLE, 0)
    da, db, home = _operands(a, b)
    c = DenseMatrix.zeros(a.rows, b.cols, a.prec, da.device)
    flag = _flag(da.device) if c.is_device else None
    _simple_into(da, db, c, threads, flag)
    return _result(_check_finite(c, flag), home)


MODES = ("exact", "fast", "tensor")


def matmul_block(a, b, n_min, threads=1, *, mode="exact", gpus=1):
    """Blocked product with block size ``n_min``; bit-identical to
    :func:`matmul_simple` at every block size (multiply.py:171-182).

    ``gpus`` (a count or a device list) > 1 row-shards C over the GPUs of
    this node with B broadcast over NCCL (north_star (5)); the result is
    bitwise the one-GPU product.

    ``mode="fast"`` (DD only) opts into the faithful 15-instruction DD
    sequence: within the north_star bound 4 l u (|A||B|)_ij (u = 2^-104) but
    NOT bit-identical to the reference.
    ``mode="tensor"`` (DD and QD) returns the exact product rounded once,
    computed on the int8 tensor cores (``tensor.py``); n_min is ignored."""
    _check_pair(a, b, threads)
    if n_min < 1:
        raise ValueError("block size must be positive")
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}; expected one of {MODES}")
    if mode == "fast" and a.prec.kind is not Kind.DD:
        raise ValueError("the fast accuracy mode is implemented for DD only")
    devs = _gpu_list(gpus)
    if len(devs) > 1:
        if mode == "tensor":
            raise ValueError("the tensor mode runs on one GPU")
        return _rows_multi(a, b, _cuda.ALGO_BLOCK_FAST if mode == "fast" else _cuda.ALGO_BLOCK,
                           n_min, devs)
    if mode == "tensor":
        if not backend.is_cuda():
            raise ValueError("the tensor mode runs on the cuda backend only")
        from .tensor import matmul_exact
        return matmul_exact(a, b)
    if backend.is_cuda() and not a.is_device and not b.is_device:
        algo = _cuda.ALGO_BLOCK_FAST if mode == "fast" else _cuda.ALGO_BLOCK
        return _host_product(a, b, algo, n_min)
    da, db, home = _operands(a, b)
    if mode == "fast":
        if not backend.is_cuda():
            raise ValueError("the fast accuracy mode runs on the cuda backend only")
        c = DenseMatrix.empty(a.rows, b.cols, a.prec, da.device)
        flag = _flag(da.device)
        _gemm_view(_cuda.ALGO_BLOCK_FAST, n_min, _View.of(da.data), _View.of(db.data),
                   _View.of(c.data), False, flag.data_ptr())
        return _result(_check_finite(c, flag), home)
    if backend.is_cuda():
        # zeros + accumulate-into == accumulate from a zero register
        # accumulator: skip the memset and start from zero in the kernel
        c = DenseMatrix.empty(a.rows, b.cols, a.prec, da.device)
        flag = _flag(da.device)
        _gemm_view(_cuda.ALGO_BLOCK, n_min, _View.of(da.data), _View.of(db.data),
                   _View.of(c.data), False, flag.data_ptr())
        return _result(_check_finite(c, flag), home)
    c = DenseMatrix.zeros(a.rows, b.cols, a.prec)
    _block_into(da, db, c, n_min, threads)
    return _result(_check_finite(c), home)


# ---------------------------------------------------------------------------
# elementwise helper (multiply.py:189-203)
# ---------------------------------------------------------------------------

def _ewise(x, y, subtract, stats=None):
    """New matrix x +/- y (one reference ewise op)."""
    if x.is_device or backend.is_cuda():
        dx, dy = x.to_device(), y.to_device(x.device)
        out = DenseMatrix.empty(x.rows, x.cols, x.prec, dx.device)
        _ewise_view(_View.of(out.data), _View.of(dx.data), _View.of(dy.data),
                    -1 if subtract else 1)
        out = out if x.is_device else out.to_host()
    else:
        out = DenseMatrix.zeros(x.rows, x.cols, x.prec)
        kern = backend.kernels()
        pre = "dd" if x.prec.kind is Kind.DD else "qd"
        getattr(kern, f"{pre}_ewise_{'sub' if subtract else 'add'}")(
            x.data, y.data, out.data, 0, x.rows)
    if stats is not None:
        stats.additions += 1
    return out


# ---------------------------------------------------------------------------
# Strassen (multiply.py:267-338), on strided device views
# ---------------------------------------------------------------------------

def matmul_strassen(a, b, cutoff=DEFAULT_STRASSEN_CUTOFF, leaf_n_min=DEFAULT_BLOCK_SIZE,
                    threads=1, stats=None, *, rectangular=False, gpus=1):
    """Seven-product recursion with the reference's semantics.

    Square inputs only unless ``rectangular=True`` (an extension for
    BASELINE config 3's 2048x1024x4096 case: each odd dimension is padded
    to even and the quadrants are m/2 x l/2 and l/2 x n/2, PAPER.md:42;
    recursion stops when the smallest dimension is <= cutoff).  For square
    inputs both modes are the reference's algorithm, bit for bit.

    ``gpus`` (a count or a device list) > 1 spreads the seven top-level
    products over the GPUs -- the reference's own parallel Strassen runs
    them on a thread pool (multiply.py:324-329) -- with the operand sums and
    the combination on the first GPU: bitwise the one-GPU recursion.
    """
    if not rectangular and not (a.rows == a.cols == b.rows == b.cols):
        raise ShapeError("Strassen requires square inputs of equal dimension")
    _check_pair(a, b, threads)
    if cutoff < 2:
        raise ValueError("Strassen cutoff must be >= 2")
    if leaf_n_min < 1:
        raise ValueError("leaf block size must be positive")
    if stats is not None and threads != 1:
        raise ValueError("operation counting is only supported for serial runs")
    if not backend.is_cuda():
        raise ValueError("Strassen runs on the cuda backend only")
    devs = _gpu_list(gpus)
    da, db, home = _operands(a, b)
    if len(devs) > 1 and min(a.rows, a.cols, b.cols) > cutoff and not rectangular:
        c = _strassen_multi(da, db, cutoff, leaf_n_min, devs, stats)
        return _result(_check_finite(c), home)
    c = DenseMatrix.empty(a.rows, b.cols, a.prec, da.device)
    _strassen_rec(_View.of(da.data), _View.of(db.data), _View.of(c.data), cutoff, leaf_n_min,
                  stats)
    return _result(_check_finite(c), home)


def _strassen_rec(A, B, C, cutoff, leaf_n_min, stats):
    """The reference's recursion (multiply.py:293-338) through the native
    driver (csrc/strassen.cpp, mpmm_strassen_dev): level-synchronous --
    per level one batched elementwise launch per operand shape, ONE batched
    GEMM launch for all 7^d leaves, one batched launch per level for the
    quadrant combinations -- with the same padding, operand list,
    combination chains and zero-accumulator leaves, so results are
    bit-identical to the reference."""
    import ctypes
    counts = (ctypes.c_int64 * 2)()
    _cuda.strassen_dev(C.comps, cutoff, leaf_n_min, A.rows, A.cols, B.cols, A.ptr, A.ld,
                       B.ptr, B.ld, C.ptr, C.ld, None, counts if stats is not None else None,
                       _stream())
    if stats is not None:
        stats.multiplications += counts[0]
        stats.additions += counts[1]


def _strassen_multi(da, db, cutoff, leaf_n_min, devs, stats):
    """The top level of the recursion with its seven products on ``devs``
    (product i on devs[i % len(devs)]): operand sums on the first device in
    the reference's order (multiply.py:313-321), each product below the top
    level by the native recursion on its device (multiply.py:293-338), the
    quadrant combination back on the first device (multiply.py:334-337).
    Per element the operations are the one-GPU recursion's: same bits."""
    import ctypes

    from . import shard
    torch = _torch()
    home = da.data.device
    prec = da.prec
    n, comps = da.rows, prec.comps
    even = n + (n & 1)
    A, B = da.data, db.data
    if even != n:   # zero padding of an odd dimension (multiply.py:293-299)
        A = torch.zeros((even, even, comps), dtype=torch.float64, device=home)
        B = torch.zeros((even, even, comps), dtype=torch.float64, device=home)
        A[:n, :n] = da.data
        B[:n, :n] = db.data
    h = even // 2

    def add(x, y, subtract):
        out = torch.empty((h, h, comps), dtype=torch.float64, device=home)
        _ewise_view(_View.of(out), _View.of(x), _View.of(y), -1 if subtract else 1)
        if stats is not None:
            stats.additions += 1
        return out

    qa = [A[i * h:(i + 1) * h, j * h:(j + 1) * h].contiguous() for i in (0, 1) for j in (0, 1)]
    qb = [B[i * h:(i + 1) * h, j * h:(j + 1) * h].contiguous() for i in (0, 1) for j in (0, 1)]
    ops = shard.strassen_operands(*qa, *qb, add)
    home_stream = torch.cuda.current_stream(home)
    ready = torch.cuda.Event()
    ready.record(home_stream)
    prods, events = [], []
    for i, (x, y) in enumerate(ops):
        dev = torch.device("cuda", devs[i % len(devs)])
        with torch.cuda.device(dev):
            s = torch.cuda.current_stream(dev)
            s.wait_event(ready)
            X, Y = x.to(dev, non_blocking=True), y.to(dev, non_blocking=True)
            P = torch.empty((h, h, comps), dtype=torch.float64, device=dev)
            counts = (ctypes.c_int64 * 2)() if stats is not None else None
            _cuda.strassen_dev(comps, cutoff, leaf_n_min, h, h, h, X.data_ptr(), h,
                               Y.data_ptr(), h, P.data_ptr(), h, None, counts, s.cuda_stream)
            if stats is not None:
                stats.multiplications += counts[0]
                stats.additions += counts[1]
            ev = torch.cuda.Event()
            ev.record(s)
            prods.append(P)
            events.append(ev)
            # the operand copies must outlive the queued product
            X.record_stream(s)
            Y.record_stream(s)
    if stats is not None:
        stats.multiplications += 7
    for ev in events:
        home_stream.wait_event(ev)
    prods = [p.to(home, non_blocking=True) for p in prods]
    c11, c12, c21, c22 = shard.strassen_combine(prods, add)
    c = torch.cat([torch.cat([c11, c12], dim=1), torch.cat([c21, c22], dim=1)], dim=0)
    return DenseMatrix(n, n, prec, c[:n, :n].contiguous())


# ---------------------------------------------------------------------------
# dispatch (multiply.py:345-350)
# ---------------------------------------------------------------------------

def run_choice(a, b, choice, threads=1, *, gpus=1):
    """Run a tuner outcome; ``gpus`` as in matmul_block / matmul_strassen."""
    if choice.kind is Algorithm.SIMPLE:
        return matmul_simple(a, b, threads, gpus=gpus)
    if choice.kind is Algorithm.BLOCK:
        return matmul_block(a, b, choice.n_min, threads, gpus=gpus)
    if choice.kind is Algorithm.EXACT:
        from .tensor import NotRepresentable, matmul_exact
        try:
            return matmul_exact(a, b)
        except NotRepresentable:
            # operands outside the int8 CRT range: the mirror blocked kernel
            return matmul_block(a, b, choice.n_min or DEFAULT_BLOCK_SIZE, threads, gpus=gpus)
    return matmul_strassen(a, b, choice.cutoff, choice.n_min, threads, gpus=gpus)
