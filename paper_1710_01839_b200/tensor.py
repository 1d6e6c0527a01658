"""Exact DD/QD products on the int8 tensor cores (opt-in "tensor" mode).

``matmul_exact(a, b)`` returns the EXACT product of the DD/QD operands,
rounded once to the nearest DD/QD expansion -- more accurate than the
reference's step-by-step rounding (so not bit-identical to it), and far
inside the north_star bound 4 l u (|A||B|)_ij.

How (csrc/ozaki.cu, int8gemm.cpp; the CRT variant of the Ozaki scheme):

1. scan (one pass per operand, one host sync): per row of A (column of
   B) and component the largest exponent E and the lowest set bit L; for a
   component range the row shift s = -min L makes every entry times 2^s an
   integer of < beta = max(E - L) + 1 (+1 per doubling of the range) bits;
2. residues: each scaled entry as a two's-complement word string, reduced
   modulo N pairwise-coprime prime powers p_t <= 256 by byte dot products
   (dp4a) with 2^(8j) mod p_t, centred into int8; N is the smallest count
   whose product P exceeds 2 l 2^(beta_A + beta_B);
3. one batched int8 GEMM per modulus (exact int32 accumulation);
4. CRT: per output, X = sum_t r_t W_t mod P rebuilt in 32-bit limbs,
   scaled by 2^-(s_i + t_j), summed over jobs, rounded to DD/QD.

When beta_A + beta_B does not fit the 54 available moduli (363 bits) the
operands are split into component ranges (e.g. QD hi/lo of A against all
of B, or hi/lo of both) and the exact jobs are summed in the combine step,
so the result stays the exact product, correctly rounded; the planner
takes the feasible split with the least int8/CRT work.  ``NotRepresentable``
is raised when even single components do not fit (e.g. a row spanning
2^300 of dynamic range).
"""

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


_dev_cache = {}


def _device_const(key, host_array, device):
    k = (key, str(device))
    if k not in _dev_cache:
        import torch
        _dev_cache[k] = torch.from_numpy(np.ascontiguousarray(host_array)).to(device)
    return _dev_cache[k]


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

    def fits(self, actual_a, actual_b):
        """The plan is exact for operands whose per-range widths are these."""
        return all(x <= y for x, y in zip(actual_a, self.beta_a)) and \
            all(x <= y for x, y in zip(actual_b, self.beta_b))

    def loose(self, actual_a, actual_b, slack=8):
        """Much wider than needed (a fresh plan would use fewer moduli)."""
        return any(x + slack < y for x, y in zip(actual_a, self.beta_a)) or \
            any(x + slack < y for x, y in zip(actual_b, self.beta_b))


_PLANS = {}   # (device, stream, comps, m, l, n) -> Plan of the last product


def _widths(raw, ranges):
    """Device betas (max(E - L) + 1 per range, 0 when empty) -> planner
    widths (+1 bit per doubling of the range's component count)."""
    return [max(int(b), 1) + (c1 - c0 - 1).bit_length() for b, (c0, c1) in zip(raw, ranges)]


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


def _execute(pl, A, B, buf, aux, ea, stream):
    """Shifts, residues, int8 GEMMs and the CRT combine for plan ``pl``;
    everything is enqueued on ``stream`` (no host sync)."""
    import torch
    m, l, comps = A.shape
    n = B.shape[1]
    dev = A.device
    pad = lambda x: -(-x // 16) * 16  # noqa: E731  (cuBLASLt IMMA alignment)
    mp_, np_, lp = pad(m), pad(n), pad(l)
    sh_a = torch.empty((len(pl.ranges_a), m), dtype=torch.int32, device=dev)
    sh_b = torch.empty((len(pl.ranges_b), n), dtype=torch.int32, device=dev)
    _cuda.oz_shifts_dev(comps, pl.ranges_a, m, buf.data_ptr(), sh_a.data_ptr(),
                        aux[1:].data_ptr(), stream)
    _cuda.oz_shifts_dev(comps, pl.ranges_b, n, buf[ea:].data_ptr(), sh_b.data_ptr(),
                        aux[5:].data_ptr(), stream)
    alloc = torch.zeros if (mp_, np_, lp) != (m, n, l) else torch.empty
    RA, RB = [], []
    for r, (c0, c1) in enumerate(pl.ranges_a):
        R = alloc((pl.need_a[r], mp_, lp), dtype=torch.int8, device=dev)
        _cuda.oz_residues_dev(0, comps, c0, c1, m, l, A.data_ptr(), A.shape[1], sh_a[r].data_ptr(),
                              pl.need_a[r], pl.words_a[r], R.data_ptr(), lp, mp_ * lp, stream)
        RA.append(R)
    for r, (c0, c1) in enumerate(pl.ranges_b):
        R = alloc((pl.need_b[r], np_, lp), dtype=torch.int8, device=dev)
        _cuda.oz_residues_dev(1, comps, c0, c1, l, n, B.data_ptr(), B.shape[1], sh_b[r].data_ptr(),
                              pl.need_b[r], pl.words_b[r], R.data_ptr(), lp, np_ * lp, stream)
        RB.append(R)
    ws = torch.empty(WORKSPACE_BYTES, dtype=torch.uint8, device=dev)
    rec = np.zeros(len(pl.jobs), dtype=_REC)
    Gs = []
    for q, (ia, ib, N) in enumerate(pl.jobs):
        G = torch.empty((N, mp_, np_), dtype=torch.int32, device=dev)
        _cuda.int8_gemm_batched_dev(mp_, np_, lp, N, RA[ia].data_ptr(), RB[ib].data_ptr(),
                                    G.data_ptr(), ws.data_ptr(), WORKSPACE_BYTES, stream)
        table = _device_const(("crt", N, pl.K), crt_table(N, pl.K)[0], dev)
        rec[q] = (G.data_ptr(), sh_a[ia].data_ptr(), sh_b[ib].data_ptr(), table.data_ptr(), N,
                  pl.K, np_, mp_ * np_)
        Gs.append(G)
    C = torch.empty((m, n, comps), dtype=torch.float64, device=dev)
    _cuda.oz_combine_dev(comps, rec.ctypes.data, len(pl.jobs), m, n, C.data_ptr(),
                         aux.data_ptr(), stream)
    # buffers return to the caching allocator in stream order
    return C


_REC = np.dtype([("G", "<u8"), ("sr", "<u8"), ("sc", "<u8"), ("tb", "<u8"), ("N", "<i4"),
                 ("K", "<i4"), ("gp", "<i8"), ("gl", "<i8")])


class _Replay:
    """The whole device side of one product (scans, shifts, residues, int8
    GEMMs, combine) captured as a CUDA graph for fixed operand addresses:
    repeated products of the same operands pay one graph launch instead of
    ~15 host-side launches.  The data are read afresh at every replay, and
    the widths it reports are checked against the plan as on the eager path."""

    def __init__(self, pl, A, B):
        import torch
        self.pl = pl
        self.ptrs = (A.data_ptr(), B.data_ptr())
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            stream = torch.cuda.current_stream().cuda_stream
            buf, aux, ea, _ = _scan(A, B, stream)
            self.C = _execute(pl, A, B, buf, aux, ea, stream)
        self.aux = aux

    def run(self):
        self.graph.replay()
        return self.aux.cpu().numpy()


_REPLAYS = {}        # key -> _Replay
_LAST_PTRS = {}      # key -> operand addresses of the previous product
GRAPH_MAX_BYTES = 1 << 30     # intermediates a cached graph may keep alive


def _graph_bytes(pl, m, l, n):
    pad = lambda x: -(-x // 16) * 16  # noqa: E731
    g = sum(N for _, _, N in pl.jobs) * pad(m) * pad(n) * 4
    r = (sum(pl.need_a) * pad(m) + sum(pl.need_b) * pad(n)) * pad(l)
    return g + r


def _check(h, pl):
    if h[0] & 1:
        raise RangeError("non-finite operand or product overflowed the working precision")
    if h[0] & 2:
        raise NotRepresentable("CRT combine window exceeded")
    return (_widths(h[1:1 + len(pl.ranges_a)], pl.ranges_a),
            _widths(h[5:5 + len(pl.ranges_b)], pl.ranges_b))


def matmul_exact_tensors(A, B):
    """C = A*B for (m,l,comps) / (l,n,comps) float64 CUDA tensors, exact
    product rounded once to comps doubles; returns the (m,n,comps) tensor.

    A product of the same shape on the same stream as the previous one
    reuses its plan speculatively: the scans, the device-side shifts and
    width check, the residues, GEMMs and combine are all enqueued at once
    and the ONE host sync reads the status and the actual widths; if the
    data needs a wider plan than the cached one the product is planned and
    recomputed (never returned wrong).  When the same operands come back
    (same addresses) the device side replays as one CUDA graph."""
    import torch
    m, l, comps = A.shape
    n = B.shape[1]
    dev = A.device
    stream = torch.cuda.current_stream(dev).cuda_stream
    key = (dev.index, stream, comps, m, l, n)
    ptrs = (A.data_ptr(), B.data_ptr())
    rp = _REPLAYS.get(key)
    if rp is not None and rp.ptrs == ptrs:
        try:
            act = _check(rp.run(), rp.pl)
            if rp.pl.fits(*act) and not rp.pl.loose(*act):
                return rp.C.clone()
        except (RangeError, NotRepresentable):
            pass                      # redo eagerly: same error, or the exact reason
        _REPLAYS.pop(key, None)
        _PLANS.pop(key, None)
    buf, aux, ea, eb = _scan(A, B, stream)
    pl = _PLANS.get(key)
    speculative = pl is not None
    if pl is None:
        pl = _make_plan(buf, ea, eb, comps, m, l, n)
    C = _execute(pl, A, B, buf, aux, ea, stream)
    h = aux.cpu().numpy()
    try:
        act_a, act_b = _check(h, pl)
    except RangeError:
        _PLANS.pop(key, None)
        raise
    if speculative and not pl.fits(act_a, act_b):
        pl = _make_plan(buf, ea, eb, comps, m, l, n)
        aux.zero_()
        C = _execute(pl, A, B, buf, aux, ea, stream)
        act_a, act_b = _check(aux.cpu().numpy(), pl)
    if pl.loose(act_a, act_b):
        _PLANS.pop(key, None)        # next product of this shape replans
        _LAST_PTRS.pop(key, None)
        return C
    _PLANS[key] = pl
    if _LAST_PTRS.get(key) == ptrs and _graph_bytes(pl, m, l, n) <= GRAPH_MAX_BYTES:
        try:
            _REPLAYS[key] = _Replay(pl, A, B)
        except RuntimeError:
            _REPLAYS.pop(key, None)   # capture not possible here: stay eager
    _LAST_PTRS[key] = ptrs
    return C


def matmul_exact(a, b):
    """DenseMatrix product through the exact tensor mode (result where ``a`` is)."""
    from .matrix import DenseMatrix
    from .multiply import _check_pair
    _check_pair(a, b, 1)
    da, db = a.to_device(), b.to_device(a.device if a.is_device else None)
    C = matmul_exact_tensors(da.data, db.data)
    c = DenseMatrix(a.rows, b.cols, a.prec, C)
    return c if a.is_device else c.to_host()
