#!/usr/bin/env python3
"""Build a variant of libmpmm_cuda.so with extra nvcc flags into a given
path (experiments; load it with MPMM_LIB_PATH).
usage: build_variant.py OUT.so [nvcc flags...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1710_01839_b200 import _build as b  # noqa: E402

out, extra = sys.argv[1], sys.argv[2:]
cmd = [b.nvcc()] + b.NVCC_FLAGS + extra + ["-o", out] + [os.path.join(b.CSRC, f) for f in b.SOURCES]
sys.exit(subprocess.run(cmd).returncode)
