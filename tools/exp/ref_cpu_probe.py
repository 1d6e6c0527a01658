"""Why the reference arm's CPU slice time depends on where B lives: times
the reference's blocked kernel (oracle/_ref) on the 128-row slice of the
8192 DD product with B in ordinary numpy memory, in mlock'ed memory, in
torch-pinned memory, and as a copy first-touched by all threads; prints the
host's NUMA layout and automatic-NUMA-balancing setting."""
import ctypes, mmap, os, subprocess, sys, time
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle
import bench

for cmd in (["lscpu"], ["numactl", "-H"]):
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=10).stdout
        print("\n".join(l for l in out.splitlines() if "NUMA" in l or "node" in l or "Model name" in l or "Socket" in l))
    except OSError as e:
        print(cmd, e)
for f in ("/proc/sys/kernel/numa_balancing", "/sys/kernel/mm/transparent_hugepage/enabled"):
    try:
        print(f, open(f).read().strip())
    except OSError as e:
        print(f, e)
inp = bench._inputs_module()
a, b = inp.gemm_inputs("dd", 8192, 8192, 8192, seed=1)
kern = oracle.ref_kernels()
cores = len(os.sched_getaffinity(0))
sl = np.ascontiguousarray(a[:128])

def t(bb, label):
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        oracle.matmul_block(sl, bb, 64, threads=cores, kernels=kern)
        ts.append(time.perf_counter() - t0)
    print(f"{label:34s} {min(ts):.2f} s  {ts}", flush=True)

def locked_copy(x):
    size = (x.nbytes + 4095) // 4096 * 4096
    mm = mmap.mmap(-1, size, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    buf = np.frombuffer(mm, dtype=np.uint8)
    libc = ctypes.CDLL("libc.so.6", use_errno=True)
    rc = libc.mlock(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(size))
    print("mlock rc", rc, ctypes.get_errno())
    out = buf[:x.nbytes].view(x.dtype).reshape(x.shape)
    out[...] = x
    return out

def parallel_touch_copy(x):
    out = np.empty_like(x)
    rows = np.array_split(np.arange(x.shape[0]), cores)
    def cp(r):
        if len(r):
            out[r[0]:r[-1] + 1] = x[r[0]:r[-1] + 1]
    with ThreadPoolExecutor(cores) as p:
        list(p.map(cp, rows))
    return out

t(b, "numpy generated")
t(locked_copy(b), "mlock'ed copy")
t(parallel_touch_copy(b), "copy first-touched by all threads")
t(bench.hugepage_copy(b), "hugepage (mmap+madvise) copy")
import torch
t(torch.from_numpy(b).pin_memory().numpy(), "torch pinned")
