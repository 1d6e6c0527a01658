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
from .errors import DeviceError


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


class PeerOperand:
    """B shared over peer memory instead of broadcast (the fused
    alternative to the NCCL broadcast; ``csrc/peer.cpp``).

    Collective: every rank of ``group`` constructs it.  The source rank
    copies its B into a buffer it exports by CUDA IPC; the handle travels
    once through ``torch.distributed``; every other rank maps the buffer.
    ``ptr`` is then B's address as this rank sees it: passed as B to the
    GEMM, the kernel reads B's tiles from the source GPU's HBM over
    NVLink/NVSwitch while it computes -- no broadcast, no k-panel schedule,
    the same kernels and therefore the same bits.  ``close()`` (collective)
    unmaps and, on the source rank after a barrier, frees."""

    def __init__(self, b, *, group=None, src=0):
        import torch.distributed as dist
        self.group, self.src = group, src
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.shape = tuple(b.shape) if b is not None else None
        self.ptr = None
        obj = [None]
        if self.rank == src:
            import torch
            torch.cuda.synchronize(b.device)      # B complete before the copy
            try:
                self.ptr, handle = _cuda.ipc_alloc(b.numel() * 8, b.data_ptr())
                obj = [(handle, self.shape)]
            except Exception as ex:  # noqa: BLE001 - every rank raises below
                obj = [("error", str(ex))]
        if dist.is_initialized():
            dist.broadcast_object_list(obj, src=_group_rank_to_global(group, src), group=group)
        if obj[0][0] == "error":
            raise DeviceError(f"peer operand: the source rank failed: {obj[0][1]}")
        handle, self.shape = obj[0]
        if self.rank != src:
            self.ptr = _cuda.ipc_open(handle)

    def close(self):
        """Collective: unmap, barrier, free on the source rank (every rank
        must call it, also one whose mapping failed)."""
        import torch.distributed as dist
        if self.ptr is not None and self.rank != self.src:
            _cuda.ipc_close(self.ptr)
        if dist.is_initialized():
            dist.barrier(group=self.group)
        if self.ptr is not None and self.rank == self.src:
            _cuda.ipc_free(self.ptr)
        self.ptr = None


def peer_matmul(a_local, peer_b, *, n_min=64, simple=False, nonfinite=None):
    """C_local = A_local * B with B read over peer memory (PeerOperand):
    one GEMM launch on this rank, its B tiles pulled from the source GPU."""
    import torch
    comps = a_local.shape[2]
    l, n = peer_b.shape[0], peer_b.shape[1]
    rows = a_local.shape[0]
    c_local = torch.empty((rows, n, comps), dtype=torch.float64, device=a_local.device)
    if rows:
        _cuda.gemm_dev(comps, _cuda.ALGO_SIMPLE if simple else _cuda.ALGO_BLOCK, n_min, rows, l,
                       n, a_local.data_ptr(), l, peer_b.ptr, n, c_local.data_ptr(), n, False,
                       nonfinite, torch.cuda.current_stream().cuda_stream)
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


# ---------------------------------------------------------------------------
# Strassen's seven top-level products spread over ranks (SURVEY.md s8f-2:
# the alternative to row sharding)
# ---------------------------------------------------------------------------

def strassen_operands(a11, a12, a21, a22, b11, b12, b21, b22, add):
    """The seven (left, right) operand pairs of the reference's recursion
    (multiply.py:300-318), in its order and with its sums; add(x, y,
    subtract) is one reference ewise op."""
    return (
        (add(a11, a22, False), add(b11, b22, False)),
        (add(a21, a22, False), b11),
        (a11, add(b12, b22, True)),
        (a22, add(b21, b11, True)),
        (add(a11, a12, False), b22),
        (add(a21, a11, True), add(b11, b12, False)),
        (add(a12, a22, True), add(b21, b22, False)),
    )


def strassen_combine(p, add):
    """C quadrants from the seven products, the reference's chains
    (multiply.py:320-331)."""
    p1, p2, p3, p4, p5, p6, p7 = p
    c11 = add(add(add(p1, p4, False), p5, True), p7, False)
    c12 = add(p3, p5, False)
    c21 = add(p2, p4, False)
    c22 = add(add(add(p1, p3, False), p2, True), p6, False)
    return c11, c12, c21, c22


def strassen_distributed(a, b, *, product, add, group=None):
    """C = A B (square, both operands on every rank, torch tensors of shape
    (n, n, comps)) with the seven top-level Strassen products computed on
    ranks i mod world: rank r forms the operand sums of its products,
    multiplies them with ``product`` (the recursion below the top level:
    matmul_strassen with the same cutoff, or the blocked kernel at a leaf),
    and each product is broadcast from its owner (the exchange step; the
    only collective).  Every rank then combines the quadrants in the
    reference's order, so C is bitwise the single-process Strassen's.
    ``add(x, y, subtract)``: one reference ewise op on same-shape tensors.
    The caller handles n <= cutoff (no top level to split)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n, comps = a.shape[0], a.shape[2]
    even = n + (n & 1)
    if even != n:   # the reference pads an odd dimension with zeros (multiply.py:293-299)
        ap = a.new_zeros((even, even, comps))
        bp = b.new_zeros((even, even, comps))
        ap[:n, :n] = a
        bp[:n, :n] = b
        a, b = ap, bp
    h = even // 2

    def q(m, i, j):
        return m[i * h:(i + 1) * h, j * h:(j + 1) * h].contiguous()

    mine = [i for i in range(7) if i % world == rank]
    # only the sums this rank's products need (the rest are never formed)
    ops = strassen_operands(q(a, 0, 0), q(a, 0, 1), q(a, 1, 0), q(a, 1, 1),
                            q(b, 0, 0), q(b, 0, 1), q(b, 1, 0), q(b, 1, 1),
                            _Lazy.add(add))
    prods = []
    for i in range(7):
        if i in mine:
            x, y = ops[i]
            prods.append(product(_Lazy.force(x), _Lazy.force(y)).contiguous())
        else:
            prods.append(a.new_empty((h, h, comps)))
    if world > 1:
        for i in range(7):
            dist.broadcast(prods[i], src=_group_rank_to_global(group, i % world), group=group)
    c11, c12, c21, c22 = strassen_combine(prods, add)
    c = torch.cat([torch.cat([c11, c12], dim=1), torch.cat([c21, c22], dim=1)], dim=0)
    return c[:n, :n].contiguous()


def _group_rank_to_global(group, r):
    import torch.distributed as dist
    if group is None:
        return r
    return dist.get_global_rank(group, r)


class _Lazy:
    """A deferred ewise op, formed only when a product needs it."""

    def __init__(self, fn, args):
        self.fn, self.args = fn, args

    @staticmethod
    def add(add):
        return lambda x, y, subtract: _Lazy(add, (x, y, subtract))

    @staticmethod
    def force(v):
        if isinstance(v, _Lazy):
            x, y, s = v.args
            return v.fn(_Lazy.force(x), _Lazy.force(y), s)
        return v


def cuda_strassen_ops(prec, cutoff, leaf_n_min):
    """(product, add) on device tensors through the sm_100a kernels: the
    product is matmul_strassen at the same cutoff (the blocked kernel when
    the half size is at or below it), add one batched ewise launch."""
    from .matrix import DenseMatrix
    from . import multiply as mul

    def product(x, y):
        X = DenseMatrix(x.shape[0], x.shape[1], prec, x)
        Y = DenseMatrix(y.shape[0], y.shape[1], prec, y)
        if x.shape[0] <= cutoff:
            return mul.matmul_block(X, Y, leaf_n_min).data
        return mul.matmul_strassen(X, Y, cutoff, leaf_n_min).data

    def add(x, y, subtract):
        X = DenseMatrix(x.shape[0], x.shape[1], prec, x)
        Y = DenseMatrix(y.shape[0], y.shape[1], prec, y)
        return mul._ewise(X, Y, subtract).data

    return product, add
