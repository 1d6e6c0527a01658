"""INTEGRATION.md option B, executed: the reference-side binding stub
(tests/integration/_kernels_cuda.py, the INTEGRATION.md code block verbatim
-- checked below) is a complete kernel module of the reference's
protocol (backend.py:28-56) over libmpmm_cuda.so.  Driven the way the
reference's multiply.py drives a backend, its results equal the oracle's
(the reference restated, pinned to its goldens) bit for bit."""

import importlib.util
import os
import re

import numpy as np
import pytest

import oracle
from paper_1710_01839_b200 import _cuda, inputs

HERE = os.path.dirname(os.path.abspath(__file__))
STUB = os.path.join(HERE, "integration", "_kernels_cuda.py")


def load_stub():
    os.environ["MPMM_CUDA_LIB"] = _cuda.LIB_PATH
    spec = importlib.util.spec_from_file_location("_kernels_cuda", STUB)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_stub_is_the_documented_binding():
    doc = open(os.path.join(os.path.dirname(HERE), "INTEGRATION.md")).read()
    m = re.search(r"```python\n(# mpmm/_kernels_cuda.py.*?)```", doc, re.S)
    assert m and m.group(1) == open(STUB).read()


@pytest.mark.gpu
@pytest.mark.parametrize("tok,shape", [("dd", (37, 45, 29)), ("qd", (13, 11, 9))])
def test_stub_protocol_bitwise(gpu, tok, shape):
    k = load_stub()
    assert k.NAME == "cuda"
    m, l, n = shape
    a, b = inputs.gemm_inputs(tok, m, l, n, seed=61)
    want = oracle.matmul_simple(a, b)
    c = np.zeros_like(want)
    getattr(k, f"{tok}_simple_rows")(a, b, c, 0, m)
    assert np.array_equal(c, want)
    for n_min in (4, 16):
        cells = (-(-m // n_min)) * (-(-n // n_min))
        c = np.zeros_like(want)
        getattr(k, f"{tok}_block_cells")(a, b, c, n_min, 0, cells // 3)
        getattr(k, f"{tok}_block_cells")(a, b, c, n_min, cells // 3, cells)
        assert np.array_equal(c, want)
    y = inputs.gemm_inputs(tok, m, l, n, seed=62)[0]
    for op, sub in (("add", False), ("sub", True)):
        out = np.zeros_like(a)
        getattr(k, f"{tok}_ewise_{op}")(a, y, out, 0, m)
        assert np.array_equal(out, oracle.ewise_new(a, y, sub))


@pytest.mark.gpu
def test_c_caller_option_c(gpu, tmp_path):
    """INTEGRATION.md option C: tests/c/abi_smoke.c, a C program using only
    include/mpmm_cuda.h, built with gcc against the in-tree library and the
    oracle, runs and matches the oracle bit for bit."""
    import subprocess
    root = os.path.dirname(HERE)
    oracle.lib()                       # builds oracle/liboracle.so if needed
    exe = str(tmp_path / "abi_smoke")
    libdir = os.path.dirname(_cuda.LIB_PATH)
    odir = os.path.join(root, "oracle")
    subprocess.run(["gcc", "-O2", "-o", exe, os.path.join(HERE, "c", "abi_smoke.c"),
                    "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
                    "-L", libdir, "-l:libmpmm_cuda.so", "-L", odir, "-l:liboracle.so",
                    "-L", "/usr/local/cuda/lib64", "-lcudart",
                    f"-Wl,-rpath,{libdir}:{odir}:/usr/local/cuda/lib64"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "abi_smoke ok" in r.stdout
