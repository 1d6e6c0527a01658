import torch, time
torch.manual_seed(0)
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / reps / 1e3
for (m, k, n) in ((1024, 1024, 1024), (4096, 1024, 1024), (33 * 1024, 1024, 1024), (8192, 8192, 8192)):
    a = torch.randint(-127, 128, (m, k), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (k, n), dtype=torch.int8, device="cuda")
    dt = t(lambda: torch._int_mm(a, b))
    print(f"int8 {m}x{k}x{n}: {dt*1e6:.1f} us  {2*m*k*n/dt/1e12:.1f} TOPS")
a = [torch.randint(-127, 128, (1024, 1024), dtype=torch.int8, device="cuda") for _ in range(33)]
b = [torch.randint(-127, 128, (1024, 1024), dtype=torch.int8, device="cuda") for _ in range(33)]
dt = t(lambda: [torch._int_mm(x, y) for x, y in zip(a, b)], 5)
print(f"33 x int8 1024^3 sequential: {dt*1e3:.3f} ms  {33*2*1024**3/dt/1e12:.1f} TOPS")
# reference check: exactness
x = a[0].int().double(); y = b[0].int().double()
print("exact:", torch.equal(torch._int_mm(a[0], b[0]).double(), x @ y))
