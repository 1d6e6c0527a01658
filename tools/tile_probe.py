#!/usr/bin/env python3
"""Time every CTA tile configuration (MPMM_FORCE_TILE) on one product and
check all of them give the same bits.  usage: tile_probe.py dd|qd n [reps]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["TILE_16", "TILE_32", "TILE_64", "TILE_32x64", "TILE_LPT"]
EXTRA = [int(x) for x in os.environ.get("PROBE_EXTRA", "").split(",") if x]

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import hashlib
    import torch
    from paper_1710_01839_b200 import _cuda, inputs
    tok, n, reps = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    comps = 2 if tok == "dd" else 4
    A, B = inputs.gemm_inputs_device(tok, n, n, n, seed=0)
    C = torch.empty((n, n, comps), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def run():
        _cuda.gemm_dev(comps, _cuda.ALGO_BLOCK, 32, n, n, n, A.data_ptr(), n, B.data_ptr(), n,
                       C.data_ptr(), n, False, None, s)
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    h = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:12]
    F = 53 if tok == "dd" else 796
    print(f"{os.environ['MPMM_FORCE_TILE']} {ts[0]:.4f} {ts[len(ts) // 2]:.4f} "
          f"{F * n ** 3 / (ts[len(ts) // 2] * 1e-3) / 1e12:.3f} {h}", flush=True)
    sys.exit(0)

tok = sys.argv[1] if len(sys.argv) > 1 else "dd"
n = sys.argv[2] if len(sys.argv) > 2 else "1024"
reps = sys.argv[3] if len(sys.argv) > 3 else "10"
hashes = set()
print(f"{tok} {n}^3: tile min_ms med_ms TFLOP/s(F) hash")
for t in list(range(len(NAMES))) + EXTRA:
    env = dict(os.environ, MPMM_FORCE_TILE=str(t))
    out = subprocess.run([sys.executable, __file__, "--child", tok, n, reps], env=env,
                         capture_output=True, text=True)
    line = out.stdout.strip() or out.stderr.strip().splitlines()[-1]
    print(f"{NAMES[t] if t < len(NAMES) else 'exp':10s} {line}", flush=True)
    if out.returncode == 0:
        hashes.add(line.split()[-1])
print("bitwise identical across tiles:", len(hashes) == 1)
