"""Pinned host<->device copy bandwidth on this box (the e2e leg's bound)."""
import torch, time
n = 38441808
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(29360128, dtype=torch.uint8).pin_memory()
d2 = torch.empty(29360128, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def timeit(f, reps=20):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / reps
t_h2d = timeit(lambda: d.copy_(h, non_blocking=True))
t_d2h = timeit(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
t_both = timeit(both)
print(f"H2D {n/t_h2d/1e9:.1f} GB/s ({t_h2d*1e3:.3f} ms for 38.4 MB); D2H {29360128/t_d2h/1e9:.1f} GB/s ({t_d2h*1e3:.3f} ms for 29.4 MB); both concurrently {t_both*1e3:.3f} ms")
