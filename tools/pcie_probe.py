"""PCIe bound of the end-to-end build: H2D of the cfg3 mesh (840 MB) and D2H of its grid
(240 MB) from/to page-locked memory, alone and concurrently (two streams)."""
import time
import torch

h_in = torch.empty(840_000_000, dtype=torch.uint8).pin_memory()
h_out = torch.empty(239_429_360, dtype=torch.uint8).pin_memory()
d_in = torch.empty_like(h_in, device="cuda")
d_out = torch.empty_like(h_out, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d(); d2h()


a, b, c = timed(h2d), timed(d2h), timed(both)
print(f"H2D 840 MB: {a:.2f} ms ({840 / a:.1f} GB/s); D2H 239 MB: {b:.2f} ms ({239.4 / b:.1f} GB/s); "
      f"both concurrently: {c:.2f} ms -> e2e bound {1e3 / c:.1f} builds/s")
