"""Exact DD/QD products on the int8 tensor cores (opt-in "tensor" mode).

``matmul_exact(a, b)`` returns the EXACT product of the DD/QD operands,
rounded once to the nearest DD/QD expansion -- more accurate than the
reference's step-by-step rounding (so not bit-identical to it), and far
inside the north_star bound 4 l u (|A||B|)_ij.

How (csrc/ozaki.cu, int8gemm.cpp; the CRT variant of the Ozaki scheme):

1. scan: per row of A (column of B) the largest exponent E and the lowest
   set bit L of any component; the row shift s = -L makes every entry
   times 2^s an integer of < beta = max(E - L) + 1 bits;
2. residues: those integers modulo N pairwise-coprime prime powers
   p_t <= 256, centred into int8, with N the smallest count whose product
   P exceeds 2 l 2^(beta_A + beta_B);
3. one batched int8 GEMM per modulus (exact int32 accumulation);
4. CRT: per output, X = sum_t r_t W_t mod P rebuilt in 32-bit limbs,
   scaled by 2^-(s_i + t_j), summed over jobs, rounded to DD/QD.

When beta_A + beta_B does not fit the 54 available moduli (363 bits) the
operands are split into component ranges (hi/lo) and the exact jobs
hi*hi + hi*lo + lo*hi + lo*lo are summed in the combine step, so the
result stays the exact product, correctly rounded.  ``NotRepresentable``
is raised when even single components do not fit (e.g. a row spanning
2^300 of dynamic range).
"""

import math
from functools import lru_cache

import numpy as np

from . import _cuda
from .errors import MpmmError, RangeError

MODULI = (256, 251, 243, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191,
          181, 179, 173, 169, 167, 163, 157, 151, 149, 139, 137, 131, 127, 125,
          121, 113, 109, 107, 103, 101, 97, 89, 83, 79, 73, 71, 67, 61,
          59, 53, 49, 47, 43, 41, 37, 31, 29, 23, 19, 17)
EMPTY_E = -100000
WORKSPACE_BYTES = 64 << 20


class NotRepresentable(MpmmError, ValueError):
    """The operands' dynamic range is too wide for the int8 CRT scheme."""


def moduli_count(bits):
    """Smallest N with prod(MODULI[:N]) > 2^bits, or None."""
    P = 1
    for n, p in enumerate(MODULI, start=1):
        P *= p
        if P > (1 << bits):
            return n
    return None


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


@lru_cache(maxsize=None)
def pow2_table(N, xmax):
    t = np.zeros((N, xmax), dtype=np.uint8)
    for i, p in enumerate(MODULI[:N]):
        t[i] = [pow(2, x, p) for x in range(xmax)]
    return t


_dev_cache = {}


def _device_const(key, host_array, device):
    k = (key, str(device))
    if k not in _dev_cache:
        import torch
        _dev_cache[k] = torch.from_numpy(np.ascontiguousarray(host_array)).to(device)
    return _dev_cache[k]


def _scan(X, rows, cols, comps, c0, c1, by_cols, stream):
    import torch
    n = cols if by_cols else rows
    E = torch.empty(n, dtype=torch.int32, device=X.device)
    L = torch.empty(n, dtype=torch.int32, device=X.device)
    _cuda.oz_scan_dev(1 if by_cols else 0, comps, c0, c1, rows, cols, X.data_ptr(),
                      X.shape[1], E.data_ptr(), L.data_ptr(), stream)
    E, L = E.cpu().numpy(), L.cpu().numpy()
    full = E != EMPTY_E
    beta = int((E[full] - L[full]).max()) + 1 if full.any() else 1
    shift = np.where(full, -L, 0).astype(np.int32)
    return beta, shift


def _split_plans(comps):
    """Component-range job lists to try, widest ranges first.  Every list
    covers all pairs, so the sum of the jobs is the exact product."""
    ranges = {2: [[(0, 2)], [(0, 1), (1, 2)]],
              4: [[(0, 4)], [(0, 2), (2, 4)], [(0, 1), (1, 2), (2, 3), (3, 4)]]}[comps]
    return [[(ra, rb) for ra in rs for rb in rs] for rs in ranges]


def plan(A, B, stream=None):
    """The job list ``[(ra, rb, N, beta_a, beta_b, shift_a, shift_b)]``."""
    import torch
    m, l, comps = A.shape
    n = B.shape[1]
    stream = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    log_l = max(1, math.ceil(math.log2(max(l, 2))))
    cache = {}
    for jobs in _split_plans(comps):
        out = []
        for ra, rb in jobs:
            if ("a", ra) not in cache:
                cache[("a", ra)] = _scan(A, m, l, comps, ra[0], ra[1], False, stream)
            if ("b", rb) not in cache:
                cache[("b", rb)] = _scan(B, l, n, comps, rb[0], rb[1], True, stream)
            ba, sa = cache[("a", ra)]
            bb, sb = cache[("b", rb)]
            N = moduli_count(ba + bb + log_l + 1)
            if N is None:
                break
            out.append((ra, rb, N, ba, bb, sa, sb))
        else:
            return out
    raise NotRepresentable("operand dynamic range too wide for the int8 CRT scheme")


def matmul_exact_tensors(A, B):
    """C = A*B for (m,l,comps) / (l,n,comps) float64 CUDA tensors, exact
    product rounded once to comps doubles; returns the (m,n,comps) tensor."""
    import torch
    m, l, comps = A.shape
    n = B.shape[1]
    if not (torch.isfinite(A).all() and torch.isfinite(B).all()):
        raise RangeError("non-finite operand: the exact tensor mode needs finite inputs")
    dev = A.device
    stream = torch.cuda.current_stream(dev).cuda_stream
    jobs = plan(A, B, stream)
    ws = torch.empty(WORKSPACE_BYTES, dtype=torch.uint8, device=dev)
    pad = lambda x: -(-x // 16) * 16  # noqa: E731  (cuBLASLt IMMA alignment)
    mp_, np_, lp = pad(m), pad(n), pad(l)
    K = max(crt_limbs(N) for _, _, N, _, _, _, _ in jobs)
    # residues once per operand component range, with the most moduli any
    # job using that range needs (a job reads the leading planes)
    need = {}
    for ra, rb, N, ba, bb, sa, sb in jobs:
        need[("a", ra)] = max(need.get(("a", ra), 0), N)
        need[("b", rb)] = max(need.get(("b", rb), 0), N)
    xmax = max(max(j[3], j[4]) for j in jobs) + 8
    res = {}
    alloc = torch.zeros if (mp_, np_, lp) != (m, n, l) else torch.empty
    for ra, rb, N, ba, bb, sa, sb in jobs:
        for side, rng, sh in (("a", ra, sa), ("b", rb, sb)):
            if (side, rng) in res:
                continue
            Nr = need[(side, rng)]
            pow2 = _device_const(("pow2", Nr, xmax), pow2_table(Nr, xmax), dev)
            dsh = torch.from_numpy(sh).to(dev)
            if side == "a":
                R = alloc((Nr, mp_, lp), dtype=torch.int8, device=dev)
                _cuda.oz_residues_dev(0, comps, rng[0], rng[1], m, l, A.data_ptr(), l,
                                      dsh.data_ptr(), Nr, pow2.data_ptr(), xmax, R.data_ptr(),
                                      lp, mp_ * lp, stream)
            else:
                R = alloc((Nr, np_, lp), dtype=torch.int8, device=dev)
                _cuda.oz_residues_dev(1, comps, rng[0], rng[1], l, n, B.data_ptr(), n,
                                      dsh.data_ptr(), Nr, pow2.data_ptr(), xmax, R.data_ptr(),
                                      lp, np_ * lp, stream)
            res[(side, rng)] = (R, dsh)
    keep, recs = [], []
    for ra, rb, N, ba, bb, sa, sb in jobs:
        RA, dsa = res[("a", ra)]
        RB, dsb = res[("b", rb)]
        table = _device_const(("crt", N, K), crt_table(N, K)[0], dev)
        G = torch.empty((N, mp_, np_), dtype=torch.int32, device=dev)
        _cuda.int8_gemm_batched_dev(mp_, np_, lp, N, RA.data_ptr(), RB.data_ptr(), G.data_ptr(),
                                    ws.data_ptr(), WORKSPACE_BYTES, stream)
        keep += [G, dsa, dsb]
        recs.append((G.data_ptr(), dsa.data_ptr(), dsb.data_ptr(), table.data_ptr(), N, K,
                     np_, mp_ * np_))
    del res
    rec = np.zeros(len(recs), dtype=np.dtype([("G", "<u8"), ("sr", "<u8"), ("sc", "<u8"),
                                              ("tb", "<u8"), ("N", "<i4"), ("K", "<i4"),
                                              ("gp", "<i8"), ("gl", "<i8")]))
    for q, r in enumerate(recs):
        rec[q] = r
    drec = torch.from_numpy(rec.view(np.uint8).copy()).to(dev)
    C = torch.empty((m, n, comps), dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _cuda.oz_combine_dev(comps, drec.data_ptr(), len(recs), m, n, C.data_ptr(),
                         status.data_ptr(), rec.ctypes.data, stream)
    st = int(status.item())
    if st & 2:
        raise NotRepresentable("CRT combine window exceeded")
    if st & 1:
        raise RangeError("matrix product overflowed the working precision")
    del keep
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
