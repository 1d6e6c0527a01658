#!/bin/bash
# Time the variant libraries built by build_variant.py (tile_probe per lib).
out=gpurun_out/variants.log
: > $out
for lib in tools/exp/qdlibs/*.so; do
  echo "== $lib" >> $out
  MPMM_LIB_PATH=$PWD/$lib timeout 300 python tools/tile_probe.py qd 1024 5 >> $out 2>&1
done
for lib in tools/exp/ddlibs/*.so; do
  echo "== $lib $(grep "$(basename $lib .so | sed 's/lib_//') " tools/exp/ddlibs/VARIANTS)" >> $out
  for n in 1024 2048; do
    MPMM_FORCE_TILE=1 MPMM_LIB_PATH=$PWD/$lib timeout 300 python - $n >> $out 2>&1 <<'PY'
import sys, os, hashlib, torch
sys.path.insert(0, os.getcwd())
from paper_1710_01839_b200 import _cuda, inputs
n = int(sys.argv[1])
A, B = inputs.gemm_inputs_device("dd", n, n, n, seed=0)
C = torch.empty((n, n, 2), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
run = lambda: _cuda.gemm_dev(2, _cuda.ALGO_BLOCK, 32, n, n, n, A.data_ptr(), n, B.data_ptr(), n, C.data_ptr(), n, False, None, s)
run(); torch.cuda.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"  dd {n}: min {ts[0]:.4f} med {ts[3]:.4f} ms  frac(F=53, 36.7T) {53*n**3/(ts[3]*1e-3)/36.7e12:.4f} hash {hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:12]}")
PY
  done
done
cat $out
