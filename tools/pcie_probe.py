"""Host<->device copy bandwidth on this box: H2D alone, D2H alone, both at once."""
import time

import torch

N = 1 << 30
dev = torch.device("cuda", 0)
h_in = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(N, dtype=torch.uint8, device=dev)
d_out = torch.empty(N, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


a = timed(h2d)
b = timed(d2h)
c = timed(both)
print(f"H2D {N / a / 1e9:.1f} GB/s  D2H {N / b / 1e9:.1f} GB/s  both: {2 * N / c / 1e9:.1f} GB/s total ({c * 1e3:.1f} ms vs {a * 1e3:.1f}+{b * 1e3:.1f})")
