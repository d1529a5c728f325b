"""PCIe bandwidth on the box: pinned H2D, D2H, and both at once (4 GB)."""
import time

import torch

n = 4_096_000_000 // 8
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def h2d():
    d_a.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_b, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


gb = n * 8 / 1e9
th, td, tb = t(h2d), t(d2h), t(both)
print(f"H2D {gb / th:.1f} GB/s  D2H {gb / td:.1f} GB/s  both at once: {gb / tb:.1f} GB/s each ({tb * 1e3:.1f} ms for "
      f"{gb:.2f} GB each way)")
