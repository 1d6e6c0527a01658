"""Exact componentwise verification on the GPU.

``exact_bound_ratio(a, b, c)`` returns, for sampled outputs (or all),

    |c_ij - (AB)_ij| / (4 l u (|A||B|)_ij)

with (AB)_ij evaluated exactly by the superaccumulator kernel
(``csrc/verify.cu``, C-ABI ``mpmm_exact_check_dev``).  Values <= 1 mean
the north_star bound holds; u = 2^-104 (DD) or 2^-209 (QD).  It is the
device-side counterpart of the Python big-integer checker used by the test
suite (``oracle/exact.py``), fast enough to check whole 1024^2 products
and large samples of 8192^2 ones.
"""

import numpy as np

from . import _cuda
from .scalar import Kind


def _sample(m, n, samples, seed):
    if samples is None or samples >= m * n:
        ii, jj = np.divmod(np.arange(m * n, dtype=np.int64), n)
        return ii, jj
    rng = np.random.default_rng(seed)
    ii = rng.integers(0, m, size=samples, dtype=np.int64)
    jj = rng.integers(0, n, size=samples, dtype=np.int64)
    ii[:4] = [0, 0, m - 1, m - 1]
    jj[:4] = [0, n - 1, 0, n - 1]
    return ii, jj


def exact_bound_ratio(a, b, c, samples=None, *, seed=0, u_exp=None):
    """``(max_ratio, ratios, (rows, cols))`` over the sampled outputs.

    ``samples``: None for every entry, an int for that many seeded random
    entries (the four corners included), or an ``(rows, cols)`` pair of
    index arrays.  NaN ratios (possible TwoProd underflow) count as failures
    in ``max_ratio`` (it becomes NaN)."""
    import torch
    if a.cols != b.rows or (c.rows, c.cols) != (a.rows, b.cols):
        raise ValueError("shape mismatch")
    comps = a.prec.comps
    if u_exp is None:
        u_exp = 104 if a.prec.kind is Kind.DD else 209
    da, db, dc = a.to_device(), b.to_device(), c.to_device()
    if isinstance(samples, tuple):
        ii, jj = (np.asarray(x, dtype=np.int64) for x in samples)
    else:
        ii, jj = _sample(a.rows, b.cols, samples, seed)
    dev = da.device
    ti = torch.from_numpy(np.ascontiguousarray(ii)).to(dev)
    tj = torch.from_numpy(np.ascontiguousarray(jj)).to(dev)
    out = torch.empty(len(ii), dtype=torch.float64, device=dev)
    _cuda.exact_check_dev(comps, a.rows, a.cols, b.cols, da.data.data_ptr(), a.cols,
                          db.data.data_ptr(), b.cols, dc.data.data_ptr(), c.cols,
                          ti.data_ptr(), tj.data_ptr(), len(ii), u_exp, out.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
    r = out.cpu().numpy()
    worst = float(np.nan) if np.isnan(r).any() else float(r.max(initial=0.0))
    return worst, r, (ii, jj)
