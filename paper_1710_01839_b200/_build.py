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
SOURCES = ["gemm_dd.cu", "gemm_qd.cu", "domain.cu", "ewise.cu", "verify.cu", "rng.cu", "ozaki.cu", "tc_i8.cu", "int8gemm.cpp",
           "strassen.cpp", "runtime.cpp", "peer.cpp", "oz_plan.cpp", "exact.cpp", "capi.cu", "host_norms.cpp"]
HEADERS = ["ddqd.cuh", "common.cuh", "kernels.h", "gemm.cuh", "domain.cuh", "trace.h"]

# -fmad=false: no implicit contraction (the reference is built with
# -ffp-contract=off, pkg/setup.py:9-11); explicit __fma_rn stays a DFMA.
COMPILE_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "-fmad=false",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
]
LINK_FLAGS = [
    "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
    "-lcublasLt", "-ldl", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
]
NVCC_FLAGS = COMPILE_FLAGS + LINK_FLAGS
OBJDIR = os.path.join(os.path.dirname(HERE), "build", "objs")


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


def _compile_one(src, obj, extra):
    cmd = [nvcc()] + COMPILE_FLAGS + list(extra) + ["-c", "-o", obj, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return cmd, r


def build(force=False, verbose=False, extra=()):
    """Compile every source to an object under build/ in parallel (one nvcc
    per file), then link the shared library."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJDIR, exist_ok=True)
    jobs = []
    for f in SOURCES:
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJDIR, os.path.splitext(f)[0] + ".o")
        jobs.append((src, obj))
    workers = max(1, min(len(jobs), os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=workers) as ex:
        results = list(ex.map(lambda j: _compile_one(j[0], j[1], extra), jobs))
    failed = False
    for cmd, r in results:
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        if r.stdout or r.stderr:
            print(r.stdout + r.stderr, file=sys.stderr)
        failed |= r.returncode != 0
    if failed:
        raise subprocess.CalledProcessError(1, "nvcc")
    cmd = [nvcc()] + LINK_FLAGS + ["-o", LIB] + [o for _, o in jobs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else ())
