#!/usr/bin/env python3
"""Build a variant of libmpmm_cuda.so with extra nvcc flags into a given
path (experiments; load it with MPMM_LIB_PATH).  Only the sources named
with --only are recompiled with the flags; the rest are linked from the
regular build's objects (build/objs).
usage: build_variant.py OUT.so [--only a.cu,b.cu] [nvcc flags...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1710_01839_b200 import _build as b  # noqa: E402

out, extra = sys.argv[1], sys.argv[2:]
only = None
if extra[:1] == ["--only"]:
    only, extra = set(extra[1].split(",")), extra[2:]
b.build()   # the regular objects
objs = []
vdir = os.path.join(os.path.dirname(os.path.abspath(out)), os.path.basename(out) + ".objs")
os.makedirs(vdir, exist_ok=True)
for f in b.SOURCES:
    base = os.path.splitext(f)[0] + ".o"
    if only is None or f in only:
        o = os.path.join(vdir, base)
        cmd = [b.nvcc()] + b.COMPILE_FLAGS + extra + ["-c", "-o", o, os.path.join(b.CSRC, f)]
        subprocess.run(cmd, check=True)
        objs.append(o)
    else:
        objs.append(os.path.join(b.OBJDIR, base))
sys.exit(subprocess.run([b.nvcc()] + b.LINK_FLAGS + ["-o", out] + objs).returncode)
