"""Host<->device copy bandwidth with pinned buffers (the e2e leg's ceiling): H2D alone, D2H
alone, both at once on two streams, and the bench step's byte counts."""
import time, torch
n = 268435456   # 256 MiB, the e2e step's H2D bytes
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def tm(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def h2d():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
def both():
    h2d(); d2h()
for name, f in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    t = tm(f)
    print(f"{name}: {t*1e3:.2f} ms  {n/t/1e9:.1f} GB/s per direction")
