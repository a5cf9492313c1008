"""Host<->device copy rates for the drop-in reindex(mesh) path (pageable numpy <-> HBM).

    python tools/hostio_probe.py [--mb 2490]

Compares the staged pinned ring of hostio (default threads / chunk), more threads, bigger
chunks, and page-locking the numpy buffer in place (cudaHostRegister) + one DMA.
"""
import argparse
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_09812_b200 import hostio  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=2490)
    a = ap.parse_args()
    n = a.mb << 20
    src = np.random.default_rng(0).integers(0, 255, size=n, dtype=np.uint8)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    print(f"host cores {os.cpu_count()}, {a.mb} MB")
    for threads in (8, 16):
        for chunk in (32, 64):
            st = hostio._Stager(chunk=chunk << 20, depth=3, threads=threads)
            t = timed(lambda: st.h2d(src, dst, s))
            print(f"staged h2d threads={threads:2d} chunk={chunk}MB: {n / t / 1e9:6.1f} GB/s ({t * 1e3:.1f} ms)")
            out = np.empty(n, dtype=np.uint8)
            t = timed(lambda: st.d2h(dst, out, s))
            print(f"staged d2h threads={threads:2d} chunk={chunk}MB: {n / t / 1e9:6.1f} GB/s ({t * 1e3:.1f} ms) (warm dst)")
    cudart = ctypes.CDLL("libcudart.so") if False else None
    # page-lock the numpy buffer in place
    from cuda.bindings import runtime as rt
    ptr = src.ctypes.data
    t0 = time.perf_counter()
    err, = rt.cudaHostRegister(ptr, n, 0)
    t_reg = time.perf_counter() - t0
    ht = torch.from_numpy(src)
    t = timed(lambda: dst.copy_(ht, non_blocking=True))
    t0 = time.perf_counter()
    rt.cudaHostUnregister(ptr)
    t_unreg = time.perf_counter() - t0
    print(f"hostRegister {t_reg * 1e3:.1f} ms ({err}), DMA {n / t / 1e9:.1f} GB/s ({t * 1e3:.1f} ms), "
          f"unregister {t_unreg * 1e3:.1f} ms")
    pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    t = timed(lambda: dst.copy_(pin, non_blocking=True))
    print(f"pinned DMA h2d {n / t / 1e9:.1f} GB/s; ", end="")
    t = timed(lambda: pin.copy_(dst, non_blocking=True))
    print(f"d2h {n / t / 1e9:.1f} GB/s")
    t0 = time.perf_counter()
    x = torch.empty(900 << 20, dtype=torch.uint8, pin_memory=True)
    print(f"fresh pinned alloc 900 MB: {(time.perf_counter() - t0) * 1e3:.1f} ms")
    del x


if __name__ == "__main__":
    main()
