"""Build libmpmm_cuda.so in-tree with nvcc for sm_100a.

The library travels to the GPU box with the repo snapshot (built .so files
are git-ignored but shipped), so nothing depends on a JIT cache.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmpmm_cuda.so")
SOURCES = ["gemm_dd.cu", "gemm_qd.cu", "ewise.cu", "verify.cu", "rng.cu", "ozaki.cu", "tc_i8.cu", "int8gemm.cpp",
           "strassen.cpp", "runtime.cpp", "oz_plan.cpp", "exact.cpp", "capi.cu", "host_norms.cpp"]
HEADERS = ["ddqd.cuh", "common.cuh", "kernels.h", "gemm.cuh", "trace.h"]

# -fmad=false: no implicit contraction (the reference is built with
# -ffp-contract=off, pkg/setup.py:9-11); explicit __fma_rn stays a DFMA.
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "-fmad=false",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math", "-shared",
    "-lcublasLt", "-ldl", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "mpmm_cuda.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False, extra=()):
    if not force and not _stale():
        return LIB
    cmd = [nvcc()] + NVCC_FLAGS + list(extra) + ["-o", LIB] + \
        [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else ())
