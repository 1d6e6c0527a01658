"""The multi-GPU schedule on CPU (no GPU): mpmm_multi_plan -- the row
blocks and k-panels csrc/runtime.cpp's mpmm_gemm_multi executes -- checked
for coverage and alignment, against shard.py's geometry, and executed with
an injected broadcast over the oracle's reference kernels: per GPU, its rows
of C accumulate panel by panel through C exactly as the reference's blocked
kernel accumulates across k blocks (_kernels.pyx:103-186), so the stitched
C is bitwise the single-product result for every GPU count and panel split
(the reference's threads-invariance contract)."""

import numpy as np
import pytest

import oracle
from paper_1710_01839_b200 import _cuda, inputs, shard


@pytest.mark.parametrize("m,l,G,panels", [(8192, 8192, 8, 0), (8192, 8192, 3, 0),
                                          (2730, 1000, 4, 0), (100, 300, 8, 5),
                                          (64, 7, 2, 0), (0, 16, 4, 0), (33, 0, 2, 3),
                                          (1, 1, 8, 9)])
def test_plan_geometry(m, l, G, panels):
    rows, ks = _cuda.multi_plan(m, l, G, panels)
    assert len(rows) == G
    assert rows == shard.row_shards(m, G, align=64)
    covered = [r for lo, hi in rows for r in range(lo, hi)]
    assert covered == list(range(m))
    for lo, hi in rows:
        assert lo % 64 == 0 or lo == m
    if l == 0:
        assert ks == []
    else:
        assert ks[0][0] == 0 and ks[-1][1] == l
        assert all(a1 == b0 for (_, a1), (b0, _) in zip(ks, ks[1:]))
        assert all(k1 > k0 for k0, k1 in ks)
        if panels > 0:
            assert len(ks) <= panels


def run_plan(a, b, G, panels, broadcast):
    """Execute mpmm_gemm_multi's schedule with the oracle kernels: GPU g
    holds its rows of A and a receive buffer for B; every panel of B is
    broadcast from GPU 0 (``broadcast(src_panel) -> copy``), then GPU g
    accumulates C_g += A_g[:, panel] * B[panel, :]."""
    m, l, n, comps = a.shape[0], a.shape[1], b.shape[1], a.shape[2]
    rows, ks = _cuda.multi_plan(m, l, G, panels)
    recv = [np.full((l, n, comps), np.nan) for _ in range(G)]
    parts = []
    for g, (r0, r1) in enumerate(rows):
        parts.append(np.zeros((r1 - r0, n, comps)))
    for k0, k1 in ks:
        for g in range(G):
            recv[g][k0:k1] = b[k0:k1] if g == 0 else broadcast(b[k0:k1])
        for g, (r0, r1) in enumerate(rows):
            if r1 == r0:
                continue
            a_panel = np.ascontiguousarray(a[r0:r1, k0:k1])
            b_panel = np.ascontiguousarray(recv[g][k0:k1])
            nm = 16
            cells = (-(-(r1 - r0) // nm)) * (-(-n // nm))
            oracle.block_cells(a_panel, b_panel, parts[g], nm, 0, cells)
    return np.concatenate(parts, axis=0), len(ks)


@pytest.mark.parametrize("tok,m,l,n,G,panels", [("dd", 200, 150, 70, 3, 4),
                                                ("dd", 130, 64, 40, 8, 0),
                                                ("qd", 70, 33, 20, 2, 3),
                                                ("dd", 65, 300, 30, 4, 0)])
def test_plan_executes_bitwise(tok, m, l, n, G, panels):
    a, b = inputs.gemm_inputs(tok, m, l, n, seed=50)
    sent = []

    def broadcast(x):          # the injected NCCL broadcast: a counted copy
        sent.append(x.nbytes)
        return x.copy()
    c, npan = run_plan(a, b, G, panels, broadcast)
    assert np.array_equal(c, oracle.matmul_simple(a, b))
    # every panel goes to every other GPU once: (G-1) * |B| bytes in total
    assert sum(sent) == (G - 1) * b.nbytes
