"""Fast pageable host <-> device copies for the numpy entry points.

``reindex(mesh)`` takes and returns ordinary numpy arrays.  A plain pageable
copy runs at ~11 GB/s host->device, and device->host into a freshly
allocated array at ~2 GB/s (the copy is single-threaded and page-faults the
destination as it goes) -- for the C2 soup that is >0.6 s around a 9 ms
re-index.  Here both directions go through a ring of pinned staging chunks:
worker threads move chunk k between the numpy array and its pinned buffer
(numpy releases the GIL; several threads also fault fresh destination pages
in parallel) while the copy engine moves chunk k+-1 over PCIe.

Small arrays (< ``MIN_BYTES``) use a plain copy.
"""
from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

MIN_BYTES = 16 << 20
CHUNK = 32 << 20
DEPTH = 3


class _Stager:
    def __init__(self, chunk: int = CHUNK, depth: int = DEPTH, threads: int | None = None):
        self.chunk = chunk
        self.depth = depth
        self.threads = threads or max(1, min(8, os.cpu_count() or 1))
        self.pool = ThreadPoolExecutor(self.threads, thread_name_prefix="rmx-stage")
        self.bufs = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(depth)]
        self.views = [b.numpy() for b in self.bufs]
        self._events = {}  # device index -> one event per buffer (an event binds to its first device)
        self.lock = threading.Lock()

    def events(self, stream: torch.cuda.Stream) -> list:
        dev = stream.device.index
        ev = self._events.get(dev)
        if ev is None:
            with torch.cuda.device(stream.device):
                ev = [torch.cuda.Event() for _ in range(self.depth)]
            self._events[dev] = ev
        return ev

    def _pcopy(self, dst: np.ndarray, src: np.ndarray) -> None:
        """dst[:] = src with the worker threads (1-D uint8 views of equal length)."""
        n = len(dst)
        parts = min(self.threads, max(1, n >> 22))  # >= 4 MB per part
        if parts == 1:
            np.copyto(dst, src)
            return
        step = (n + parts - 1) // parts
        futs = [self.pool.submit(np.copyto, dst[a:a + step], src[a:a + step]) for a in range(0, n, step)]
        for f in futs:
            f.result()

    def h2d(self, src: np.ndarray, dst: torch.Tensor, stream: torch.cuda.Stream) -> None:
        s = src.reshape(-1).view(np.uint8)
        d = dst.view(-1).view(torch.uint8)
        n = s.shape[0]
        with self.lock, torch.cuda.stream(stream):
            events = self.events(stream)
            used = [False] * self.depth
            for k, off in enumerate(range(0, n, self.chunk)):
                i = k % self.depth
                m = min(self.chunk, n - off)
                if used[i]:
                    events[i].synchronize()  # the copy engine is done with this buffer
                self._pcopy(self.views[i][:m], s[off:off + m])
                d[off:off + m].copy_(self.bufs[i][:m], non_blocking=True)
                events[i].record(stream)
                used[i] = True
            stream.synchronize()  # the caller may free or reuse `src` right away

    def d2h(self, src: torch.Tensor, dst: np.ndarray, stream: torch.cuda.Stream) -> None:
        s = src.reshape(-1).view(torch.uint8)
        d = dst.reshape(-1).view(np.uint8)
        n = d.shape[0]
        with self.lock, torch.cuda.stream(stream):
            events = self.events(stream)
            pending = []  # (buffer, offset, length) whose copy-in is in flight
            for k, off in enumerate(range(0, n, self.chunk)):
                i = k % self.depth
                m = min(self.chunk, n - off)
                if len(pending) == self.depth:  # this buffer is next to drain: drain it first
                    self._drain(pending.pop(0), d, events)
                self.bufs[i][:m].copy_(s[off:off + m], non_blocking=True)
                events[i].record(stream)
                pending.append((i, off, m))
            for item in pending:
                self._drain(item, d, events)

    def _drain(self, item, d: np.ndarray, events: list) -> None:
        i, off, m = item
        events[i].synchronize()
        self._pcopy(d[off:off + m], self.views[i][:m])


_stager = None
_stager_lock = threading.Lock()


def _get() -> _Stager:
    global _stager
    if _stager is None:
        with _stager_lock:
            if _stager is None:
                _stager = _Stager()
    return _stager


def to_device(src: np.ndarray, dst: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
    """dst (device, same byte size) <- src (C-contiguous host array)."""
    if src.nbytes < MIN_BYTES:
        from .pipeline import host_tensor
        d = dst.view(-1).view(torch.uint8)
        if stream is None:
            d.copy_(host_tensor(src.reshape(-1).view(np.uint8)))
        else:
            with torch.cuda.stream(stream):
                d.copy_(host_tensor(src.reshape(-1).view(np.uint8)))
        return
    _get().h2d(src, dst, stream or torch.cuda.current_stream(dst.device))


def to_host(src: torch.Tensor, dst: np.ndarray | None = None, stream: torch.cuda.Stream | None = None) -> np.ndarray:
    """Host copy of a contiguous device tensor (into ``dst`` if given), as a numpy array of the same dtype."""
    src = src.contiguous()
    if src.numel() * src.element_size() < MIN_BYTES and dst is None:
        if stream is None:
            return src.cpu().numpy()
        with torch.cuda.stream(stream):
            return src.cpu().numpy()
    if dst is None:
        dst = np.empty(tuple(src.shape), dtype=torch.empty(0, dtype=src.dtype).numpy().dtype)
    if src.numel() * src.element_size() < MIN_BYTES:
        dst[...] = src.cpu().numpy()
        return dst
    _get().d2h(src, dst, stream or torch.cuda.current_stream(src.device))
    return dst


__all__ = ["to_device", "to_host", "MIN_BYTES"]
