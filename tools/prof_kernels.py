#!/usr/bin/env python3
"""Launch one GEMM configuration a few times (for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1710_01839_b200 import _cuda, inputs  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--prec", default="dd")
    p.add_argument("--n", type=int, default=1024)
    p.add_argument("--nmin", type=int, default=64)
    p.add_argument("--simple", action="store_true")
    p.add_argument("--fast", action="store_true")
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    comps = 2 if a.prec == "dd" else 4
    x, y = inputs.gemm_inputs(a.prec, a.n, a.n, a.n, seed=0)
    A, B = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    C = torch.empty_like(A)
    algo = (_cuda.ALGO_SIMPLE if a.simple else
            _cuda.ALGO_BLOCK_FAST if a.fast else _cuda.ALGO_BLOCK)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(a.reps):
        _cuda.gemm_dev(comps, algo, a.nmin, a.n, a.n, a.n, A.data_ptr(), a.n, B.data_ptr(), a.n,
                       C.data_ptr(), a.n, False, None, s)
    torch.cuda.synchronize()
    print("ok", a)


if __name__ == "__main__":
    main()
