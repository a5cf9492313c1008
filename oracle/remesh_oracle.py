"""CPU oracle for the re-indexing hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The shipped package
(``paper_2109_09812_b200``) never imports anything under ``oracle/``; when
its CUDA library is missing it raises instead of falling back here.

It is a numpy restatement of ``remeshx.reindex`` (reference
``pkg/src/remeshx/pipeline.py:133-157``) and of the primitives it leans on
(``pkg/src/remeshx/primitives.py:16-69``).  Every function cites the
reference lines it follows.  All vertex arithmetic runs on ``uint32`` views
of the float32 words (``mesh.py:91-94``), so ``-0.0 != +0.0`` and NaN
payloads compare bitwise.

Parity pin: ``tests/test_oracle.py`` checks this module against golden
vectors produced by importing the reference itself
(``tools/make_golden.py`` -> ``tests/golden/*.npz``) and against the
reference's own known-answer tests (worked example, ``test_pipeline.py``).

The worker-pool chunking of ``parallel.py:42-59`` is reproduced for the CPU
baseline so the timed port uses the same host threads as the reference.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# reference parallel.py:18 -- below this many items the pool is not used
_POOL_MIN = 1 << 17
_U32_LIMIT = 1 << 32          # mesh.py:17 (MAX_VERTICES)


class OracleIndexError(ValueError):
    """Out-of-range element index (reference: InvalidMeshError, mesh.py:24-33)."""

    def __init__(self, issues):
        self.issues = issues
        super().__init__(f"{len(issues)} out-of-range index(es)")


def host_threads() -> int:
    """Worker count resolution of parallel.py:27-39 (env REMESHX_THREADS, else all cores)."""
    raw = os.environ.get("REMESHX_THREADS", "").strip()
    try:
        n = int(raw) if raw else 0
    except ValueError:
        n = 0
    return n if n > 0 else (os.cpu_count() or 1)


def _chunked(n: int, fn, threads: int | None) -> None:
    """Fixed partition of range(n) run on a pool (parallel.py:42-59)."""
    if n <= 0:
        return
    t = host_threads() if threads is None else max(1, int(threads))
    if t == 1 or n < _POOL_MIN:
        fn(0, n)
        return
    width = (n + t - 1) // t
    spans = [(a, min(a + width, n)) for a in range(0, n, width)]
    with ThreadPoolExecutor(max_workers=len(spans)) as ex:
        for fut in [ex.submit(fn, a, b) for a, b in spans]:
            fut.result()


def as_bits(vertices) -> np.ndarray:
    """(V, D) uint32 words of a float32 vertex array (mesh.py:91-94)."""
    arr = np.ascontiguousarray(vertices)
    if arr.dtype == np.uint32:
        return arr
    return np.ascontiguousarray(arr, dtype=np.float32).view(np.uint32)


def find_out_of_range(elements: np.ndarray, n_vertices: int) -> list[tuple[int, int, int]]:
    """(element, slot, index) triples for every bad index (mesh.py:97-100)."""
    hits = np.argwhere(elements >= n_vertices)
    return [(int(e), int(s), int(elements[e, s])) for e, s in hits]


def used_flags(elements: np.ndarray, n_vertices: int, threads=None) -> np.ndarray:
    """isUsed[v] = some element references v (pipeline.py:41-51)."""
    flat = np.ascontiguousarray(elements, dtype=np.uint32).ravel()
    flags = np.zeros(n_vertices, dtype=bool)

    def mark(a, b):
        flags[flat[a:b]] = True

    _chunked(flat.size, mark, threads)
    return flags


def cleaned_bits(bits: np.ndarray, flags: np.ndarray, repl_row: np.ndarray) -> np.ndarray:
    """Unused rows replaced by the replacement row (pipeline.py:54-63, 148)."""
    out = np.array(bits, dtype=np.uint32, copy=True)
    out[~flags] = repl_row
    return out


def lexi_order(bits: np.ndarray) -> np.ndarray:
    """Stable order, component 0 most significant, raw unsigned bits (primitives.py:23-27).

    ``np.lexsort`` sorts by its LAST key first, so the components are handed
    over in reverse: this is exactly the reference's ordering.
    """
    bits = np.atleast_2d(bits)
    if bits.shape[0] == 0:
        return np.empty(0, dtype=np.uint32)
    cols = tuple(bits[:, c] for c in range(bits.shape[1] - 1, -1, -1))
    return np.lexsort(cols).astype(np.uint32)


def head_flags(sorted_bits: np.ndarray, threads=None) -> np.ndarray:
    """nodup[i] = i == 0 or row i differs from row i-1 (pipeline.py:72-83)."""
    n = sorted_bits.shape[0]
    heads = np.ones(n, dtype=bool)
    if n < 2:
        return heads

    def cmp(a, b):
        heads[a + 1:b + 1] = (sorted_bits[a + 1:b + 1] != sorted_bits[a:b]).any(axis=1)

    _chunked(n - 1, cmp, threads)
    return heads


def compacted_ranks(heads: np.ndarray) -> tuple[np.ndarray, int]:
    """newIdx = inclusive_scan(nodup) - 1 and the unique count (pipeline.py:86-94,
    primitives.py:43-48; 64-bit accumulator, 32-bit result)."""
    if heads.size == 0:
        return np.empty(0, dtype=np.uint32), 0
    if not heads[0]:
        raise ValueError("first sorted row must be a head")
    run = np.cumsum(heads, dtype=np.int64)
    total = int(run[-1])
    if total >= _U32_LIMIT:
        raise OverflowError(f"scan total {total} outside 32-bit range")
    return (run - 1).astype(np.uint32), total


def inverse_of(order: np.ndarray) -> np.ndarray:
    """perm[order[i]] = i, with the coverage checks of pipeline.py:103-113."""
    n = order.size
    inv = np.full(n, n, dtype=np.uint64)
    if n:
        if int(order.max()) >= n:
            raise ValueError("not a permutation (entry out of range)")
        inv[order] = np.arange(n, dtype=np.uint64)
        if int(inv.max()) >= n:
            raise ValueError("not a permutation (repeated entries)")
    return inv.astype(np.uint32)


def reindex(vertices, elements, threads=None) -> dict:
    """Full pipeline of pipeline.py:133-157 on host arrays.

    Returns a dict with ``vertices`` (float32, U x D), ``elements`` (uint32,
    E x K) and the scratch fields ``is_used``, ``org_id``, ``nodup``,
    ``new_idx``, ``perm``, ``new_count`` (pipeline.py:24-38).
    """
    bits = as_bits(vertices)
    if bits.ndim != 2:
        raise ValueError("vertices must be (n, dim)")
    elements = np.ascontiguousarray(elements, dtype=np.uint32)
    if elements.ndim != 2:
        raise ValueError("elements must be (m, arity)")
    n_vtx, dim = bits.shape
    n_elem, arity = elements.shape
    if elements.size and int(elements.max()) >= n_vtx:          # mesh.py:103-105
        raise OracleIndexError(find_out_of_range(elements, n_vtx))

    flags = used_flags(elements, n_vtx, threads)
    if n_elem == 0:                                              # pipeline.py:142-146
        e32 = np.empty(0, np.uint32)
        return dict(vertices=np.empty((0, dim), np.float32),
                    elements=np.empty((0, arity), np.uint32),
                    is_used=flags, org_id=e32, nodup=np.empty(0, bool),
                    new_idx=e32, perm=e32, new_count=0)

    repl = bits[int(elements[0, 0])].copy()                      # pipeline.py:148
    clean = cleaned_bits(bits, flags, repl)
    order = lexi_order(clean)                                    # primitives.py:30-40
    sorted_bits = clean[order]
    heads = head_flags(sorted_bits, threads)
    ranks, count = compacted_ranks(heads)
    uniq = np.empty((count, dim), dtype=np.uint32)               # primitives.py:51-69
    uniq[ranks[heads]] = sorted_bits[heads]
    inv = inverse_of(order)
    out_elems = np.empty_like(elements)

    def remap(a, b):                                             # pipeline.py:116-130
        out_elems[a:b] = ranks[inv[elements[a:b]]]

    _chunked(n_elem, remap, threads)
    return dict(vertices=uniq.view(np.float32), elements=out_elems,
                is_used=flags, org_id=order, nodup=heads, new_idx=ranks,
                perm=inv, new_count=count)


def closed_form(vertices, elements) -> tuple[np.ndarray, np.ndarray]:
    """Output-only restatement used to cross-check ``reindex``.

    The output is the bitwise-sorted unique set of *used* rows and every index
    becomes the rank of its row among them.
    """
    bits = as_bits(vertices)
    elements = np.ascontiguousarray(elements, dtype=np.uint32)
    if elements.size == 0:
        return np.empty((0, bits.shape[1]), np.float32), elements.copy()
    used_rows = bits[np.unique(elements.ravel())]
    order = lexi_order(used_rows)
    srt = used_rows[order]
    keep = np.ones(len(srt), bool)
    keep[1:] = (srt[1:] != srt[:-1]).any(axis=1)
    uniq = srt[keep]
    # rank of every used row: position of its run in the sorted unique array
    run_id = np.cumsum(keep) - 1
    rank_of_used = np.empty(len(srt), np.uint32)
    rank_of_used[order] = run_id
    lut = np.zeros(bits.shape[0], np.uint32)
    lut[np.unique(elements.ravel())] = rank_of_used
    return uniq.view(np.float32), lut[elements]
