"""Row-sharded multi-GPU product with B broadcast over NCCL.

The reference parallelises by giving each thread a disjoint range of
output rows/cells (multiply.py:86-112).  Lifted to GPUs, each rank (one
process per GPU, ``torch.distributed`` over NCCL) owns a contiguous block
of C's rows and the matching rows of A, and receives all of B from the
source rank.  That broadcast is the only collective.

The broadcast is pipelined with the arithmetic: B is sent in k-panels on a
communication stream, and as panel p lands the compute stream runs
``C_local += A_local[:, panel p] * B[panel p, :]`` (panel 0 starts the
accumulator from zero).  Each element's k loop still runs in ascending
order through an accumulator that is exactly the DD/QD value stored in C,
so the result is bitwise identical to the single-GPU product for every
GPU count and panel size -- the reference's threads-invariance contract
 extended to GPUs.

``local_gemm`` is injectable so the partition/broadcast/accumulate logic
can be exercised on CPU ranks over ``gloo`` (tests/test_shard_gloo.py).
"""

import math

from . import _cuda


def row_shards(m, world, align=1):
    """Contiguous [lo, hi) row blocks, one per rank, ``ceil(m/world)`` rows
    each rounded up to ``align`` (the kernel tile height); trailing ranks
    may get fewer or zero rows."""
    if world < 1 or m < 0 or align < 1:
        raise ValueError("bad shard request")
    per = math.ceil(math.ceil(m / world) / align) * align if m else 0
    out = []
    for r in range(world):
        lo = min(m, r * per)
        hi = min(m, lo + per)
        out.append((lo, hi))
    return out


def panel_bounds(l, panel_rows):
    if panel_rows is None or panel_rows <= 0 or panel_rows >= l:
        return [(0, l)]
    return [(k0, min(l, k0 + panel_rows)) for k0 in range(0, l, panel_rows)]


def cuda_local_gemm(comps, algo, n_min):
    """The default per-panel compute: our sm_100a kernels on raw views."""
    import torch

    def run(a_local, b_panel, c_local, k0, k1, accumulate):
        m, l = a_local.shape[0], a_local.shape[1]
        n = b_panel.shape[1]
        if m == 0:
            return
        a_ptr = a_local.data_ptr() + 8 * comps * k0
        _cuda.gemm_dev(comps, algo, n_min, m, k1 - k0, n, a_ptr, l, b_panel.data_ptr(), n,
                       c_local.data_ptr(), n, accumulate, None,
                       torch.cuda.current_stream().cuda_stream)
    return run


def broadcast_matmul(a_local, b, *, n_min=64, simple=False, group=None, src=0,
                     panel_rows=None, local_gemm=None):
    """C_local = A_local * B with B broadcast from ``src`` in k-panels.

    ``a_local``: this rank's (rows, l, comps) float64 tensor; ``b``: the
    (l, n, comps) tensor -- holding B on ``src`` and a receive buffer of the
    same shape elsewhere.  Returns this rank's (rows, n, comps) C block.
    """
    import torch
    import torch.distributed as dist

    comps = a_local.shape[2]
    l, n = b.shape[0], b.shape[1]
    rows = a_local.shape[0]
    device = a_local.device
    c_local = torch.empty((rows, n, comps), dtype=torch.float64, device=device)
    panels = panel_bounds(l, panel_rows)
    if local_gemm is None:
        local_gemm = cuda_local_gemm(comps, _cuda.ALGO_SIMPLE if simple else _cuda.ALGO_BLOCK,
                                     n_min)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1 and device.type == "cuda":
        # nothing to receive: run the panels back to back on this stream
        for p, (k0, k1) in enumerate(panels):
            local_gemm(a_local, b[k0:k1], c_local, k0, k1, p > 0)
        return c_local
    if device.type != "cuda":
        for p, (k0, k1) in enumerate(panels):
            if world > 1:
                dist.broadcast(b[k0:k1], src=src, group=group)
            local_gemm(a_local, b[k0:k1], c_local, k0, k1, p > 0)
        return c_local

    compute = torch.cuda.current_stream(device)
    comm = torch.cuda.Stream(device=device)
    comm.wait_stream(compute)
    landed = []
    with torch.cuda.stream(comm):
        for k0, k1 in panels:
            if world > 1:
                dist.broadcast(b[k0:k1], src=src, group=group)
            ev = torch.cuda.Event()
            ev.record(comm)
            landed.append(ev)
    for p, (k0, k1) in enumerate(panels):
        compute.wait_event(landed[p])
        local_gemm(a_local, b[k0:k1], c_local, k0, k1, p > 0)
    b.record_stream(comm)
    return c_local


def sharded_matmul_host(a_rows, b, l, n, prec, *, n_min=64, simple=False, group=None, src=0,
                        panel_rows=None):
    """Multi-GPU product with HOST buffers, one call per rank.

    ``a_rows``: this rank's rows of A as a (rows, l, comps) numpy array;
    ``b``: the (l, n, comps) numpy B on ``src`` (``None`` elsewhere).
    Copies A's rows (and B on ``src``) to this rank's GPU, broadcasts B in
    k-panels, multiplies, checks finiteness (reference multiply.py:124-127)
    and returns this rank's C rows on the host.
    """
    import numpy as np
    import torch

    from .errors import RangeError

    dev = torch.device("cuda", torch.cuda.current_device())
    comps = prec.comps
    A = torch.from_numpy(np.ascontiguousarray(a_rows)).to(dev, non_blocking=True)
    if b is not None:
        B = torch.from_numpy(np.ascontiguousarray(b)).to(dev, non_blocking=True)
    else:
        B = torch.empty((l, n, comps), dtype=torch.float64, device=dev)
    C = broadcast_matmul(A, B, n_min=n_min, simple=simple, group=group, src=src,
                         panel_rows=panel_rows)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    if C.shape[0]:
        _cuda.nonfinite_dev(comps, C.shape[0], n, C.data_ptr(), n, flag.data_ptr(),
                            torch.cuda.current_stream().cuda_stream)
    out = C.cpu().numpy()
    if flag.item():
        raise RangeError("matrix product overflowed the working precision")
    return out
