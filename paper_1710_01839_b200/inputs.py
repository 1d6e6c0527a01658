"""Seeded synthetic inputs for the BASELINE.json configs.

BASELINE.json names no public dataset; every config draws synthetic
matrices from ``numpy.random.default_rng(seed)`` (PCG64, bit-reproducible
across hosts):

* DD (configs 0, 1, 3, 4): ``hi = U(-1,1)``, ``f = U(-1,1)``,
  ``lo = hi * 2^-53 * f``, then ``(hi, lo) = TwoSum(hi, lo)``.  Draw order:
  A's hi, A's f, then B's hi, B's f.
* wide-exponent DD (config 1, second set): after A and B, draw
  ``kA = integers(-30, 31, (m, l))`` and ``kB = integers(-30, 31, (l, n))``
  from the same stream and scale both components by ``2^k`` (exact).
* QD (config 2): ``x0 = U(-1,1)``, ``x_i = x0 * 2^(-53 i) * U(-1,1)``
  (i = 1..3), then each element is renormalised with the exact operation
  sequence of the reference's ``ddqd._compress4`` (ddqd.py:175-193),
  vectorised here.

The arrays are the reference's AoS layout ``(rows, cols, comps)`` float64.
"""

import numpy as np

_TWO_M53 = 2.0 ** -53


def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _quick_two_sum(a, b):
    s = a + b
    return s, b - (s - a)


def dd_random(rng, rows, cols):
    hi = rng.uniform(-1.0, 1.0, (rows, cols))
    f = rng.uniform(-1.0, 1.0, (rows, cols))
    lo = hi * _TWO_M53 * f
    hi, lo = _two_sum(hi, lo)
    return np.ascontiguousarray(np.stack([hi, lo], axis=-1))


def _renorm5_vec(x0, x1, x2, x3, x4):
    """Vectorised ddqd._renorm5 (ddqd.py:140-172), branch-free selects."""
    s, x4 = _quick_two_sum(x3, x4)
    s, x3 = _quick_two_sum(x2, s)
    s, x2 = _quick_two_sum(x1, s)
    s, x1 = _quick_two_sum(x0, s)
    out = np.zeros(x0.shape + (4,))
    k = np.zeros(x0.shape, dtype=np.int64)
    acc = s
    for t in (x1, x2, x3, x4):
        full = k == 3
        s_new = acc + t
        e = t - (s_new - acc)
        emit = (~full) & (e != 0.0)
        for q in range(3):
            sel = emit & (k == q)
            out[..., q] = np.where(sel, s_new, out[..., q])
        acc = np.where(emit, e, s_new)
        k = k + emit
    for q in range(4):
        out[..., q] = np.where(k == q, acc, out[..., q])
    return out


def _compress4_dense_vec(v):
    """Vectorised ddqd._compress4 for term vectors with NO zero entries."""
    v = [x.copy() for x in v]
    n = len(v)
    for _ in range(4):
        s = v[0]
        for i in range(1, n):
            s, v[i - 1] = _two_sum(s, v[i])
        v[n - 1] = s
    z = np.zeros_like(v[0])
    if n <= 4:
        w = [z] * (4 - n) + v
        return _renorm5_vec(w[3], w[2], w[1], w[0], z)
    tail = z
    for i in range(n - 4):
        tail = tail + v[i]
    return _renorm5_vec(v[n - 1], v[n - 2], v[n - 3], v[n - 4], tail)


def _compress4_scalar(terms):
    """Scalar ddqd._compress4 for the (rare) elements with zero terms."""
    v = [t for t in terms if t != 0.0]
    n = len(v)
    if n == 0:
        return (0.0, 0.0, 0.0, 0.0)
    for _ in range(4):
        s = v[0]
        for i in range(1, n):
            s, v[i - 1] = _two_sum(s, v[i])
        v[n - 1] = s
    if n <= 4:
        w = [0.0] * (4 - n) + v
        args = (w[3], w[2], w[1], w[0], 0.0)
    else:
        tail = 0.0
        for i in range(n - 4):
            tail += v[i]
        args = (v[n - 1], v[n - 2], v[n - 3], v[n - 4], tail)
    r = _renorm5_vec(*[np.array(x) for x in args])
    return tuple(float(x) for x in r)


def qd_random(rng, rows, cols):
    x0 = rng.uniform(-1.0, 1.0, (rows, cols))
    limbs = [x0]
    for i in range(1, 4):
        limbs.append(x0 * (2.0 ** (-53 * i)) * rng.uniform(-1.0, 1.0, (rows, cols)))
    out = _compress4_dense_vec(limbs)
    zero = np.zeros((rows, cols), dtype=bool)
    for x in limbs:
        zero |= x == 0.0
    for i, j in zip(*np.nonzero(zero)):
        out[i, j] = _compress4_scalar([x[i, j] for x in limbs])
    return np.ascontiguousarray(out)


def gemm_inputs(prec_token, m, l, n, seed=0, wide=False):
    """A (m, l, comps) and B (l, n, comps) for a config; see module doc."""
    rng = np.random.default_rng(seed)
    if prec_token == "dd":
        a = dd_random(rng, m, l)
        b = dd_random(rng, l, n)
        if wide:
            ka = rng.integers(-30, 31, (m, l))
            kb = rng.integers(-30, 31, (l, n))
            a = np.ldexp(a, ka[..., None])
            b = np.ldexp(b, kb[..., None])
        return a, b
    if prec_token == "qd":
        if wide:
            raise ValueError("the wide-exponent set is defined for DD only")
        return qd_random(rng, m, l), qd_random(rng, l, n)
    raise ValueError(f"unsupported precision {prec_token!r}")


def gemm_inputs_device(prec_token, m, l, n, seed=0, wide=False, device=None):
    """The same A and B as :func:`gemm_inputs`, generated in HBM
    (``csrc/rng.cu``: PCG64 jump-ahead + the numpy operation order), as
    float64 CUDA tensors of shape (rows, cols, comps).  Bitwise equal to the
    host generator (tests/test_gpu_inputs.py)."""
    import torch

    from . import _cuda
    comps = {"dd": 2, "qd": 4}[prec_token]
    if wide and prec_token != "dd":
        raise ValueError("the wide-exponent set is defined for DD only")
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    rng = np.random.default_rng(seed)
    st = rng.bit_generator.state["state"]
    a = torch.empty((m, l, comps), dtype=torch.float64, device=dev)
    b = torch.empty((l, n, comps), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _cuda.gen_inputs_dev(comps, st["state"], st["inc"], 0, m, l, a.data_ptr(), stream)
    _cuda.gen_inputs_dev(comps, st["state"], st["inc"], comps * m * l, l, n, b.data_ptr(),
                         stream)
    if wide:
        rng.bit_generator.advance(comps * (m * l + l * n))
        ka = rng.integers(-30, 31, (m, l))
        kb = rng.integers(-30, 31, (l, n))
        a.mul_(torch.from_numpy(np.ldexp(1.0, ka)).to(dev)[..., None])
        b.mul_(torch.from_numpy(np.ldexp(1.0, kb)).to(dev)[..., None])
    return a, b
