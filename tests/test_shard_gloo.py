"""Multi-rank sharding on CPU: world_size 2 over gloo.

Each rank owns a row block of A and C; B is broadcast from rank 0 in
k-panels; the per-panel compute is injected (the CPU oracle here, the
sm_100a kernels in production).  The gathered C must be bitwise equal to
the single-process product for every panel size: the GPU-count
invariance contract.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import oracle
from paper_1710_01839_b200 import inputs, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_local_gemm(a_local, b_panel, c_local, k0, k1, accumulate):
    a = a_local.numpy()[:, k0:k1].copy()
    b = b_panel.numpy().copy()
    c = c_local.numpy()
    if not accumulate:
        c[...] = 0.0
    # block_cells accumulates into c over all cells: C += A_panel B_panel
    cells = (-(-a.shape[0] // 8)) * (-(-b.shape[1] // 8)) if a.shape[0] else 0
    if cells:
        oracle.block_cells(a, b, c, 8, 0, cells)


def _worker(rank, world, port, tok, m, l, n, panel, out_path, align=4):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = inputs.gemm_inputs(tok, m, l, n, seed=5)
        lo, hi = shard.row_shards(m, world, align=align)[rank]
        a_local = torch.from_numpy(np.ascontiguousarray(a[lo:hi]))
        b_buf = torch.from_numpy(b.copy()) if rank == 0 else torch.zeros(b.shape, dtype=torch.float64)
        c_local = shard.broadcast_matmul(a_local, b_buf, panel_rows=panel, src=0,
                                         local_gemm=_oracle_local_gemm)
        np.save(f"{out_path}.{rank}.npy", c_local.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tok,m,l,n,panel", [("dd", 21, 17, 9, 5), ("dd", 16, 16, 16, None),
                                              ("qd", 7, 6, 5, 4)])
def test_two_rank_broadcast_matmul_is_bitwise_invariant(tmp_path, tok, m, l, n, panel):
    world = 2
    out = str(tmp_path / "c")
    tmp.spawn(_worker, args=(world, _free_port(), tok, m, l, n, panel, out), nprocs=world,
              join=True)
    parts = [np.load(f"{out}.{r}.npy") for r in range(world)]
    c = np.concatenate(parts, axis=0)
    a, b = inputs.gemm_inputs(tok, m, l, n, seed=5)
    assert np.array_equal(c, oracle.matmul_simple(a, b))


def test_four_ranks_uneven_64_row_shards(tmp_path):
    """World size 4 with the production 64-row alignment and m not a
    multiple of it (m = 200: shards of 64, 64, 64 and 8 rows), B in five
    uneven k-panels: the stitched C is bitwise the single product."""
    world, m, l, n = 4, 200, 150, 40
    assert [hi - lo for lo, hi in shard.row_shards(m, world, align=64)] == [64, 64, 64, 8]
    out = str(tmp_path / "c4")
    tmp.spawn(_worker, args=(world, _free_port(), "dd", m, l, n, 32, out, 64), nprocs=world,
              join=True)
    c = np.concatenate([np.load(f"{out}.{r}.npy") for r in range(world)], axis=0)
    a, b = inputs.gemm_inputs("dd", m, l, n, seed=5)
    assert np.array_equal(c, oracle.matmul_simple(a, b))


# ---------------------------------------------------------------------------
# Strassen's seven top-level products spread over ranks
# ---------------------------------------------------------------------------

def _oracle_strassen_ops(cutoff, leaf):
    def product(x, y):
        return torch.from_numpy(oracle.strassen(x.numpy(), y.numpy(), cutoff, leaf))

    def add(x, y, subtract):
        return torch.from_numpy(oracle.ewise_new(np.ascontiguousarray(x.numpy()),
                                                 np.ascontiguousarray(y.numpy()), subtract))
    return product, add


def _strassen_worker(rank, world, port, tok, n, cutoff, leaf, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = inputs.gemm_inputs(tok, n, n, n, seed=8)
        product, add = _oracle_strassen_ops(cutoff, leaf)
        c = shard.strassen_distributed(torch.from_numpy(a), torch.from_numpy(b),
                                       product=product, add=add)
        np.save(f"{out_path}.{rank}.npy", c.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,tok,n,cutoff", [(2, "dd", 24, 6), (3, "dd", 17, 4),
                                                (2, "qd", 10, 3)])
def test_strassen_products_over_ranks_bitwise(tmp_path, world, tok, n, cutoff):
    """Every rank's C equals the single-process Strassen (the reference's
    recursion restated in the oracle), bit for bit, for even and odd n."""
    out = str(tmp_path / "s")
    tmp.spawn(_strassen_worker, args=(world, _free_port(), tok, n, cutoff, 4, out), nprocs=world,
              join=True)
    a, b = inputs.gemm_inputs(tok, n, n, n, seed=8)
    want = oracle.strassen(a, b, cutoff, 4)
    for r in range(world):
        assert np.array_equal(np.load(f"{out}.{r}.npy"), want)


def test_strassen_operand_and_combine_order():
    """strassen_operands / strassen_combine reproduce the oracle's top level
    (the reference's operand sums and combination chains)."""
    a, b = inputs.gemm_inputs("dd", 8, 8, 8, seed=3)
    product, add = _oracle_strassen_ops(4, 2)   # the recursion below: same cutoff
    A, B = torch.from_numpy(a), torch.from_numpy(b)
    q = lambda m, i, j: m[i * 4:(i + 1) * 4, j * 4:(j + 1) * 4].contiguous()
    ops = shard.strassen_operands(q(A, 0, 0), q(A, 0, 1), q(A, 1, 0), q(A, 1, 1),
                                  q(B, 0, 0), q(B, 0, 1), q(B, 1, 0), q(B, 1, 1), add)
    quads = shard.strassen_combine([product(x, y) for x, y in ops], add)
    c = torch.cat([torch.cat(quads[:2], dim=1), torch.cat(quads[2:], dim=1)], dim=0)
    assert np.array_equal(c.numpy(), oracle.strassen(a, b, 4, 2))
