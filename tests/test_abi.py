"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute without a GPU)."""

import ctypes
import glob
import os
import re

import numpy as np

from conftest import ROOT, golden
from paper_1710_01839_b200 import _cuda, frobenius_norm, frobenius_rel_diff
from paper_1710_01839_b200.matrix import DenseMatrix
from paper_1710_01839_b200.scalar import PrecisionSpec


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(mpmm_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_built_for_sm100a():
    assert os.path.exists(_cuda.LIB_PATH)
    lib = _cuda.load()
    assert lib.mpmm_abi_version() == 1


def test_every_declared_symbol_is_exported_and_bound():
    lib = ctypes.CDLL(_cuda.LIB_PATH)
    declared = declared_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_cuda.exported_symbols())


def test_no_device_is_not_an_error():
    assert _cuda.device_count() >= 0


def test_tile_mapping():
    tiles = [_cuda.tile_for_nmin(n)[0] for n in (16, 32, 64, 128, 256)]
    assert len(set(tiles)) == 5        # every BASELINE n_min is a distinct tile
    assert _cuda.tile_for_nmin(1) == _cuda.tile_for_nmin(16)
    try:
        _cuda.tile_for_nmin(0)
    except ValueError:
        pass
    else:
        raise AssertionError("n_min=0 accepted")


def test_host_norms_match_reference():
    # values computed by the reference's matrix.py:229-294 (golden)
    for name, prec in (("dd_strassen_pair33_c8_l4", PrecisionSpec.dd()),
                       ("qd_strassen_pair11_c4_l4", PrecisionSpec.qd())):
        g = golden(name)
        n = g["a"].shape[0]
        A = DenseMatrix(n, n, prec, g["a"])
        B = DenseMatrix(n, n, prec, g["b"])
        CS = DenseMatrix(n, n, prec, g["c_strassen"])
        CP = DenseMatrix(n, n, prec, g["c_simple"])
        assert frobenius_norm(A) == g["norms"][0]
        assert frobenius_rel_diff(CS, CP) == g["norms"][1]
        assert frobenius_rel_diff(A, B) == g["norms"][2]


def test_symbols_in_binary_are_sm100a():
    # cuobjdump lists the embedded cubin architectures
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        return
    out = subprocess.run([tool, "--list-elf", _cuda.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
