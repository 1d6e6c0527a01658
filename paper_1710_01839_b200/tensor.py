"""Exact DD/QD products on the int8 tensor cores (opt-in "tensor" mode).

``matmul_exact(a, b)`` returns the EXACT product of the DD/QD operands,
rounded once to the nearest DD/QD expansion -- more accurate than the
reference's step-by-step rounding (so not bit-identical to it), and far
inside the north_star bound 4 l u (|A||B|)_ij.

How (csrc/ozaki.cu, tc_i8.cu, exact.cpp; the CRT variant of the Ozaki
scheme):

1. scan (one pass per operand, one host sync): per row of A (column of
   B) and component the largest exponent E and the lowest set bit L; for a
   component range the row shift s = -min L makes every entry times 2^s an
   integer of < beta = max(E - L) + 1 (+1 per doubling of the range) bits;
2. residues: each scaled entry as a two's-complement word string, reduced
   modulo N pairwise-coprime prime powers p_t <= 256 by byte dot products
   (dp4a) with 2^(8j) mod p_t, centred into int8; N is the smallest count
   whose product P exceeds 2 l 2^(beta_A + beta_B);
3. one int8 GEMM per modulus (exact int32 accumulation), hand-written on
   tcgen05 (TMA, TMEM accumulators), reduced mod p_t in its epilogue to
   bytes (cuBLASLt int32 products as the fallback);
4. CRT: per output, X = sum_t r_t W_t mod P rebuilt in 32-bit limbs (the
   sums as a u8 tensor-core product of residues and weight-limb bytes),
   scaled by 2^-(s_i + t_j), summed over jobs, rounded to DD/QD.

When beta_A + beta_B does not fit the 54 available moduli (363 bits) the
operands are split into component ranges (e.g. QD hi/lo of A against all
of B, or hi/lo of both) and the exact jobs are summed in the combine step,
so the result stays the exact product, correctly rounded; the planner
takes the feasible split with the least int8/CRT work.  ``NotRepresentable``
is raised when even single components do not fit (e.g. a row spanning
2^300 of dynamic range).
"""

import collections
import threading
from functools import lru_cache

import numpy as np

from . import _cuda
from .errors import MpmmError, RangeError

MODULI = (256, 251, 243, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191,
          181, 179, 173, 169, 167, 163, 157, 151, 149, 139, 137, 131, 127, 125,
          121, 113, 109, 107, 103, 101, 97, 89, 83, 79, 73, 71, 67, 61,
          59, 53, 49, 47, 43, 41, 37, 31, 29, 23, 19, 17)
EMPTY_E, EMPTY_L = -100000, 100000
WORKSPACE_BYTES = 64 << 20


class NotRepresentable(MpmmError, ValueError):
    """The operands' dynamic range is too wide for the int8 CRT scheme."""


@lru_cache(maxsize=None)
def moduli_count(bits):
    """Smallest N with prod(MODULI[:N]) > 2^bits, or None."""
    P = 1
    for n, p in enumerate(MODULI, start=1):
        P *= p
        if P > (1 << bits):
            return n
    return None


@lru_cache(maxsize=None)
def crt_limbs(N):
    P = 1
    for p in MODULI[:N]:
        P *= p
    return (P.bit_length() + 31) // 32


@lru_cache(maxsize=None)
def crt_table(N, K=None):
    """uint32 limbs: P (K limbs) then the N CRT weights W_t = M_t (M_t^-1 mod p_t) mod P
    (K defaults to the limbs P needs; a larger K zero-pads every entry)."""
    P = 1
    for p in MODULI[:N]:
        P *= p
    K = K or crt_limbs(N)
    words = []

    def limbs(x):
        return [(x >> (32 * q)) & 0xffffffff for q in range(K)]
    words += limbs(P)
    for p in MODULI[:N]:
        M = P // p
        W = (M * pow(M % p, -1, p)) % P
        words += limbs(W)
    return np.array(words, dtype=np.uint32), K


class Plan:
    """A chosen component split: ranges of A and B with their bit widths
    (beta) and residue word counts, and the jobs (pairs of ranges) with
    their moduli counts N and one CRT limb count K."""

    def __init__(self, jobs, ranges_a, ranges_b):
        self.ranges_a = [tuple(int(c) for c in r) for r in ranges_a]
        self.ranges_b = [tuple(int(c) for c in r) for r in ranges_b]
        self.jobs = [(int(j[0]), int(j[1]), int(j[2])) for j in jobs]   # (ia, ib, N)
        self.K = int(jobs[0][3])
        na, nb = len(self.ranges_a), len(self.ranges_b)
        self.words_a, self.words_b = [0] * na, [0] * nb
        self.beta_a, self.beta_b = [0] * na, [0] * nb
        self.need_a, self.need_b = [0] * na, [0] * nb
        for j in jobs:
            ia, ib, N = int(j[0]), int(j[1]), int(j[2])
            self.words_a[ia], self.words_b[ib] = int(j[4]), int(j[5])
            self.beta_a[ia], self.beta_b[ib] = int(j[6]), int(j[7])
            self.need_a[ia] = max(self.need_a[ia], N)
            self.need_b[ib] = max(self.need_b[ib], N)


def _scan(A, B, stream):
    """One scan per operand into a single int32 buffer: EL_A | EL_B | aux,
    aux = [status, beta_a[4], beta_b[4]] (zeroed)."""
    import torch
    m, l, comps = A.shape
    n = B.shape[1]
    ea, eb = 2 * comps * m, 2 * comps * n
    buf = torch.empty(ea + eb + 9, dtype=torch.int32, device=A.device)
    aux = buf[ea + eb:]
    aux.zero_()
    _cuda.oz_scan_dev(0, comps, m, l, A.data_ptr(), A.shape[1], buf.data_ptr(), aux.data_ptr(),
                      stream)
    _cuda.oz_scan_dev(1, comps, l, n, B.data_ptr(), B.shape[1], buf[ea:].data_ptr(),
                      aux.data_ptr(), stream)
    return buf, aux, ea, eb


def _make_plan(buf, ea, eb, comps, m, l, n):
    host = buf.cpu().numpy()                       # the host sync of a planned call
    if host[ea + eb] & 1:
        raise RangeError("non-finite operand: the exact tensor mode needs finite inputs")
    out = _cuda.oz_plan(comps, m, n, l, host[:ea], host[ea:ea + eb])
    if out is None:
        raise NotRepresentable("operand dynamic range too wide for the int8 CRT scheme")
    jobs, ra, _, rb, _ = out
    return Plan(jobs, ra, rb)


def plan(A, B, stream=None):
    """Scan both operands and plan the product (one host sync); returns a
    :class:`Plan`."""
    import torch
    stream = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    m, l, comps = A.shape
    buf, _, ea, eb = _scan(A, B, stream)
    return _make_plan(buf, ea, eb, comps, m, l, B.shape[1])


def matmul_exact_tensors(A, B):
    """C = A*B for (m,l,comps) / (l,n,comps) float64 CUDA tensors, exact
    product rounded once to comps doubles; returns the (m,n,comps) tensor.

    One call into the native driver (csrc/exact.cpp, mpmm_gemm_exact_dev):
    scans, [plan on the first product of a shape on this stream], shifts,
    residues, int8 GEMMs and the CRT combine, with the plan reused
    speculatively (device-side width check, replanned when it does not
    fit), intermediates cached, and the whole device side replayed as one
    CUDA graph when the same operand/result addresses come back."""
    import torch
    m, l, comps = A.shape
    n = B.shape[1]
    if not (A.is_contiguous() and B.is_contiguous()):
        A, B = A.contiguous(), B.contiguous()
    dev = A.device
    stream = torch.cuda.current_stream(dev).cuda_stream
    C = _out_buffer(m, n, comps, dev, stream)
    rc = _cuda.gemm_exact_dev(comps, m, l, n, A.data_ptr(), l, B.data_ptr(), n, C.data_ptr(), n,
                              stream)
    if rc == 5:
        raise RangeError(_cuda.last_error())
    if rc == 4:
        raise NotRepresentable(_cuda.last_error())
    return C.clone()


# (device, stream, shape) -> the driver's output buffer (a stable address),
# least recently used first; at most _OUT_KEEP shapes are kept
_OUT = collections.OrderedDict()
_OUT_KEEP = 4
_OUT_LOCK = threading.Lock()


def _out_buffer(m, n, comps, dev, stream):
    """A stable result address per shape and stream, so repeated products
    of the same operands can replay the driver's captured graph; callers
    get a copy.  Bounded: the least recently used shape is dropped."""
    import torch
    key = (dev.index, stream, m, n, comps, threading.get_ident())
    with _OUT_LOCK:
        buf = _OUT.pop(key, None)
        if buf is None:
            buf = torch.empty((m, n, comps), dtype=torch.float64, device=dev)
        _OUT[key] = buf
        while len(_OUT) > _OUT_KEEP:
            _OUT.popitem(last=False)
    return buf


def release():
    """Free the exact mode's cached state: result buffers here, plans,
    workspaces, graphs and pinned buffers in the native driver
    (mpmm_exact_release; entries in use by another thread are kept)."""
    with _OUT_LOCK:
        _OUT.clear()
    _cuda.exact_release()


def matmul_exact(a, b):
    """DenseMatrix product through the exact tensor mode (result where ``a`` is)."""
    from .matrix import DenseMatrix
    from .multiply import _check_pair
    _check_pair(a, b, 1)
    da, db = a.to_device(), b.to_device(a.device if a.is_device else None)
    C = matmul_exact_tensors(da.data, db.data)
    c = DenseMatrix(a.rows, b.cols, a.prec, C)
    return c if a.is_device else c.to_host()
