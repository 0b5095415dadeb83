"""Pinned host <-> device copy bandwidth: H2D, D2H, and both concurrently."""
import time

import torch

n = 1 << 30  # 1 GiB
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d_in.copy_(h_in, non_blocking=True)
    h_out.copy_(d_out, non_blocking=True)
torch.cuda.synchronize()


def t(fn, reps=4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D {n / a / 1e9:.1f} GB/s  D2H {n / b / 1e9:.1f} GB/s  concurrent {2 * n / c / 1e9:.1f} GB/s total "
      f"({n / c / 1e9:.1f} each)")
