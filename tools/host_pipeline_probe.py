#!/usr/bin/env python3
"""Time mpmm_gemm_host (host buffers in, host result out) per k-panel count."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, time
sys.path.insert(0, os.environ["ROOT"])
import torch, numpy as np
from paper_1710_01839_b200 import _cuda, inputs
n = int(os.environ.get("N", "1024"))
a, b = inputs.gemm_inputs("dd", n, n, n, seed=0)
pa = torch.from_numpy(a).pin_memory().numpy(); pb = torch.from_numpy(b).pin_memory().numpy()
pc = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
for _ in range(3):
    _cuda.gemm_host(2, 1, 32, pa, pb, pc)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); _cuda.gemm_host(2, 1, 32, pa, pb, pc); ts.append(time.perf_counter() - t0)
ts.sort()
print(f"panels={os.environ.get('MPMM_HOST_PANELS')} n={n} min={ts[0]*1e3:.3f}ms med={ts[5]*1e3:.3f}ms")
'''
for panels in ("1", "2", "4", "8"):
    env = dict(os.environ, ROOT=ROOT, MPMM_HOST_PANELS=panels)
    subprocess.run([sys.executable, "-c", CHILD], env=env, check=True)
