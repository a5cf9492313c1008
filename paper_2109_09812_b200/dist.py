"""Multi-GPU re-indexing: one mesh partitioned across the GPUs of one box.

Semantics: the G ranks together hold ONE mesh -- rank r owns a contiguous block
of vertices and the elements that reference them (local indices) -- exactly
like ``remeshx.merge`` (ops.py:10-35) concatenates meshes: the result equals
``reindex(merge([shard_0, ..., shard_{G-1}]))`` bit for bit.  Every rank gets
its slice of the global (bitwise-sorted) unique vertex array, the slice's
global offset, the global count, and its elements remapped to global indices.

Algorithm (a sample sort on deduplicated keys):

1. local re-index on each GPU (the full single-GPU CUDA pipeline): duplicates
   inside a shard disappear before anything crosses NVLink (a soup shrinks ~6x);
2. regular samples of the local sorted unique keys -> AllGather -> G-1 splitters
   (key-only splitters are balanced here: after step 1 a key occurs at most
   once per rank, so no heavy hitter survives);
3. ``rmx_lower_bound_rows`` partitions each sorted key array into G contiguous
   ranges -> all-to-all of the keys (counts first, then data);
4. each rank merges what it received -- G sorted, duplicate-free runs -- into
   the sorted unique keys of its range plus the rank of every received key
   (``rmx_merge_unique_runs``: pairwise merge-path rounds + one compaction; no
   re-sort; keys wider than 8 words are re-indexed instead).  All copies of a
   key go to the same rank, so there are no boundary duplicates;
5. AllGather of the per-rank unique counts -> global offsets;
6. reverse all-to-all of the global ids, in the order the keys arrived: each
   sender gets the global id of every local unique key back in its own sorted
   order, i.e. its old->new map, with no scatter;
7. ``rmx_gather_u32`` remaps the local elements.

Collectives go through a small ``Comm`` interface: :class:`SymmComm` (GPUs:
the data exchange as ``rmx_scatter_rows`` stores into the peers' symmetric
buffers over NVLink, the small collectives on NCCL), :class:`TorchComm`
(torch.distributed all-to-all -- NCCL, or gloo on CPU) or :class:`ThreadComm`
(G ranks as threads of one process, for tests on one GPU or on CPU).  The local steps go through a backend: :class:`CudaBackend` is the
product; tests may inject a CPU backend.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass

import torch

from . import _native
from .mesh import MeshError


# ---------------------------------------------------------------------------
# collectives
class Comm:
    """Collectives of one rank.  Every method is called by all ranks in the same order; the ones
    that return host values cost one host round trip each (reindex_distributed makes five)."""

    rank: int
    size: int

    def all_gather_ints(self, values: list[int]) -> list[list[int]]:
        """Every rank's small integer vector (same length on all ranks)."""
        raise NotImplementedError

    def all_gather_fixed(self, t: torch.Tensor) -> torch.Tensor:
        """Concatenation of every rank's ``t`` (same shape on all ranks); no host round trip."""
        raise NotImplementedError

    def count_matrix(self, send_counts: torch.Tensor) -> list[list[int]]:
        """C[s][g] = rows rank s sends to rank g, from every rank's (G,) int64 count tensor."""
        raise NotImplementedError

    def all_to_all(self, t: torch.Tensor, send_counts: list[int], C: list[list[int]] | None = None,
                   bounds: torch.Tensor | None = None) -> tuple[torch.Tensor, list[int]]:
        """Rows [sum(send_counts[:g]), sum(send_counts[:g+1])) of ``t`` to rank g; with the count
        matrix ``C`` known the counts are not exchanged again.  ``bounds`` optionally holds the
        (G+1,) int64 send bounds on the device (no host copy needed)."""
        raise NotImplementedError

    # derived
    def all_gather_int(self, x: int) -> list[int]:
        return [v[0] for v in self.all_gather_ints([int(x)])]

    def all_gather_rows(self, t: torch.Tensor) -> torch.Tensor:
        sizes = self.all_gather_int(t.shape[0])
        cap = max(sizes) if sizes else 0
        if cap == 0:
            return t.new_empty((0,) + tuple(t.shape[1:]))
        pad = t.new_zeros((cap,) + tuple(t.shape[1:]))
        pad[: t.shape[0]] = t
        every = self.all_gather_fixed(pad)
        return torch.cat([every[g * cap:g * cap + n] for g, n in enumerate(sizes)])


class TorchComm(Comm):
    """torch.distributed collectives (NCCL for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, group=None, device: torch.device | None = None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.device = device or torch.device("cpu")

    def _gather_tensor(self, t: torch.Tensor) -> torch.Tensor:
        out = t.new_empty((self.size,) + tuple(t.shape))
        if self.device.type == "cuda":
            self.dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        else:  # gloo: list form
            parts = [torch.empty_like(t) for _ in range(self.size)]
            self.dist.all_gather(parts, t.contiguous(), group=self.group)
            out = torch.stack(parts)
        return out

    def all_gather_ints(self, values: list[int]) -> list[list[int]]:
        t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=self.device)
        return [[int(x) for x in row] for row in self._gather_tensor(t).tolist()]

    def all_gather_fixed(self, t: torch.Tensor) -> torch.Tensor:
        g = self._gather_tensor(t)
        return g.reshape((self.size * t.shape[0],) + tuple(t.shape[1:]))

    def count_matrix(self, send_counts: torch.Tensor) -> list[list[int]]:
        sc = send_counts.to(device=self.device, dtype=torch.int64)
        return [[int(x) for x in row] for row in self._gather_tensor(sc).tolist()]

    def all_gather_ints_dev(self, t: torch.Tensor) -> list[list[int]]:
        """all_gather_ints of a small int64 device tensor without reading it on the host first."""
        g = self._gather_tensor(t.to(device=self.device, dtype=torch.int64).reshape(-1))
        return [[int(x) for x in row] for row in g.tolist()]

    def all_to_all(self, t, send_counts, C=None, bounds=None):
        if C is None:
            C = self.count_matrix(torch.tensor(list(send_counts), dtype=torch.int64))
        recv_counts = [C[s][self.rank] for s in range(self.size)]
        out = t.new_empty((sum(recv_counts),) + tuple(t.shape[1:]))
        self.dist.all_to_all_single(out, t.contiguous(), output_split_sizes=recv_counts,
                                    input_split_sizes=list(send_counts), group=self.group)
        return out, recv_counts


class SymmComm(TorchComm):
    """TorchComm whose all-to-all moves the rows over peer memory.

    Small collectives (counts, samples, sizes) stay on torch.distributed
    (NCCL).  The data exchange writes each rank's partition straight into the
    receivers' symmetric buffers (``torch.distributed._symmetric_memory``,
    CUDA IPC over NVLink) with ``rmx_scatter_rows``: the partition and the
    transfer are one kernel, with no send staging and no NCCL kernel
    ("B200-native fused variant").  Two device-side
    barriers per exchange order it: one before writing (every receiver has
    consumed the previous exchange: it reads the received rows before its next
    exchange on the same stream), one after (all writes have landed).  The
    returned tensor is a VIEW of the receive buffer, valid until this rank's
    next exchange.
    """

    def __init__(self, group=None, device: torch.device | None = None):
        super().__init__(group, device)
        import torch.distributed._symmetric_memory as symm
        self.symm = symm
        self.group_name = (group if group is not None else self.dist.group.WORLD).group_name
        self.lib = _native.lib()
        self._buf = None
        self._handle = None
        self._cap = 0  # int32 words

    def _ensure(self, words: int) -> None:
        """Collective: every rank calls it with the same ``words``."""
        if words <= self._cap:
            return
        cap = max(words, int(self._cap * 1.5), 1 << 16)
        buf = self.symm.empty(cap, dtype=torch.int32, device=self.device)
        self._handle = self.symm.rendezvous(buf, self.group_name)
        self._buf = buf
        self._cap = cap

    def all_to_all(self, t, send_counts, C=None, bounds=None):
        G, me = self.size, self.rank
        if t.dtype != torch.int32:
            raise MeshError("SymmComm exchanges int32 rows")
        words = 1
        for x in t.shape[1:]:
            words *= int(x)
        if C is None:
            C = self.count_matrix(torch.tensor(list(send_counts), dtype=torch.int64))
        recv_counts = [C[s][me] for s in range(G)]
        recv_total = sum(recv_counts)
        self._ensure(max(sum(C[s][g] for s in range(G)) for g in range(G)) * words)
        dst_off = [sum(C[s][g] for s in range(me)) for g in range(G)]
        if bounds is None:
            b = [0]
            for c in send_counts:
                b.append(b[-1] + c)
            meta = torch.tensor(b + dst_off, dtype=torch.int64, device=self.device)
        else:
            meta = torch.cat([bounds.to(device=self.device, dtype=torch.int64),
                              torch.tensor(dst_off, dtype=torch.int64, device=self.device)])
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self._handle.barrier(channel=0)
        n = t.shape[0]
        if n:
            src = t.contiguous()
            _native.check(self.lib.rmx_scatter_rows(src.data_ptr(), n, words, meta.data_ptr(), G,
                                                    self._handle.buffer_ptrs_dev, meta.data_ptr() + 8 * (G + 1),
                                                    stream))
        self._handle.barrier(channel=0)
        out = self._buf[:recv_total * words].view((recv_total,) + tuple(t.shape[1:]))
        return out, recv_counts


class ThreadHub:
    """Shared state of G in-process ranks (see :class:`ThreadComm`)."""

    def __init__(self, size: int):
        self.size = size
        self.slots: list = [None] * size
        self.barrier = threading.Barrier(size)


class ThreadComm(Comm):
    """G ranks as threads of one process: collectives are hand-offs through a hub.

    Used to run the multi-rank host logic on one GPU (each thread drives the
    same device) or on CPU; no rank ever waits on another inside a kernel.
    """

    def __init__(self, hub: ThreadHub, rank: int):
        self.hub = hub
        self.rank = rank
        self.size = hub.size

    def _exchange(self, obj):
        self.hub.slots[self.rank] = obj
        self.hub.barrier.wait()
        out = list(self.hub.slots)
        self.hub.barrier.wait()
        return out

    def all_gather_ints(self, values: list[int]) -> list[list[int]]:
        return [[int(x) for x in v] for v in self._exchange([int(x) for x in values])]

    def all_gather_fixed(self, t: torch.Tensor) -> torch.Tensor:
        parts = self._exchange(t)
        return torch.cat([p.to(t.device) for p in parts])

    def count_matrix(self, send_counts: torch.Tensor) -> list[list[int]]:
        return [[int(x) for x in v] for v in self._exchange([int(x) for x in send_counts.reshape(-1).tolist()])]

    def all_to_all(self, t, send_counts, C=None, bounds=None):
        parts = self._exchange((t, list(send_counts)))
        chunks, recv_counts = [], []
        for src, counts in parts:
            start = sum(counts[: self.rank])
            n = counts[self.rank]
            chunks.append(src[start:start + n].to(t.device))
            recv_counts.append(n)
        out = torch.cat(chunks) if chunks else t.new_empty((0,) + tuple(t.shape[1:]))
        return out, recv_counts


# ---------------------------------------------------------------------------
# local steps
class CudaBackend:
    """Local steps on this rank's GPU through the C-ABI."""

    def __init__(self, device: torch.device | None = None):
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.lib = _native.lib()

    def reindex(self, vertex_bits: torch.Tensor, elements: torch.Tensor):
        from .pipeline import reindex_tensors
        res = reindex_tensors(vertex_bits, elements)
        return res.vertices, res.elements

    def merge_unique(self, keys: torch.Tensor, run_counts: list[int]):
        """Sorted unique keys of G sorted duplicate-free runs + the rank of every row
        (``rmx_merge_unique_runs``: pairwise merge-path rounds, then one compaction).  Returns the
        key buffer (n rows, the first `count` valid), the ranks and the count as a device tensor:
        the caller learns the count together with the other ranks' (one round trip)."""
        import ctypes
        n, D = keys.shape
        dev = self.device
        out = torch.empty((n, D), dtype=torch.int32, device=dev)
        rank_of = torch.empty(n, dtype=torch.int32, device=dev)
        count = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = torch.empty(max(1, int(self.lib.rmx_merge_workspace_bytes(n, D))), dtype=torch.uint8, device=dev)
        starts, acc = [], 0
        for c in run_counts:
            starts.append(acc)
            acc += c
        arr = (ctypes.c_uint64 * max(1, len(starts)))(*starts)
        _native.check(self.lib.rmx_merge_unique_runs(keys.contiguous().data_ptr() if n else None, n, D, arr,
                                                     len(starts), out.data_ptr(), rank_of.data_ptr(),
                                                     count.data_ptr(), ws.data_ptr(), ws.numel(),
                                                     torch.cuda.current_stream(dev).cuda_stream))
        return out, rank_of.view(n, 1), count

    def lower_bound(self, rows: torch.Tensor, queries: torch.Tensor) -> torch.Tensor:
        """First row >= each query (rows sorted): an int64 device tensor (no host copy)."""
        q = queries.shape[0]
        out = torch.empty(q, dtype=torch.int64, device=self.device)
        if q == 0:
            return out
        rows = rows.contiguous()
        queries = queries.contiguous()
        _native.check(self.lib.rmx_lower_bound_rows(
            rows.data_ptr() if rows.numel() else None, rows.shape[0], rows.shape[1], queries.data_ptr(), q,
            out.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream))
        return out

    def gather(self, table: torch.Tensor, idx: torch.Tensor, status: torch.Tensor | None = None) -> torch.Tensor:
        """out = table[idx]; an index past the table sets ``status`` (checked by the caller when it
        wants to: the indices come from this pipeline, so it is an internal invariant)."""
        n = idx.numel()
        out = torch.empty(n, dtype=torch.int32, device=self.device)
        if n == 0:
            return out
        if status is None:
            status = torch.zeros(1, dtype=torch.int32, device=self.device)
        _native.check(self.lib.rmx_gather_u32(
            table.data_ptr() if table.numel() else None, table.numel(), idx.contiguous().data_ptr(), n,
            out.data_ptr(), status.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream))
        return out


@dataclass
class DistResult:
    """This rank's part of the distributed result.

    ``vertices``: (u_r, D) int32 bit view, the slice [offset, offset + u_r) of the
    global sorted unique vertex array; ``elements``: this rank's elements with
    GLOBAL new indices; ``total``: the global unique count.
    """

    vertices: torch.Tensor
    offset: int
    total: int
    elements: torch.Tensor


def reindex_distributed(vertex_bits: torch.Tensor, elements: torch.Tensor, comm: Comm, backend=None,
                        samples_per_rank: int = 1024, timing: dict | None = None,
                        check: bool = False) -> DistResult:
    """Re-index the mesh whose rank-r shard is (vertex_bits, elements); see module doc.

    Host round trips: the local unique count, the sample sizes, the sorted samples' count, the
    exchange count matrix, the merged counts (five, whatever G).  ``timing`` (a dict, GPU backends)
    receives CUDA-event milliseconds of the steps and the exchanged bytes; ``check`` verifies the
    internal remap indices (one more round trip).
    """
    backend = backend or CudaBackend(vertex_bits.device)
    if vertex_bits.dim() != 2 or elements.dim() != 2:
        raise MeshError("vertex_bits must be (V, D) and elements (E, K)")
    D = vertex_bits.shape[1]
    G, me = comm.size, comm.rank
    cuda = vertex_bits.is_cuda and timing is not None
    ev = {}

    def mark(name):
        if cuda:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            ev[name] = e

    mark("start")
    # 1. local dedup: sorted unique keys + local old->new indices
    uniq, local_out = backend.reindex(vertex_bits, elements)
    u = uniq.shape[0]
    mark("local")
    if G == 1:
        if cuda:
            torch.cuda.current_stream(vertex_bits.device).synchronize()
            timing["local_ms"] = ev["start"].elapsed_time(ev["local"])
        return DistResult(uniq, 0, u, local_out)
    # 2. splitters from regular samples: S rows per rank (zero-padded), the valid counts and dims
    #    gathered once
    S = max(1, samples_per_rank)
    s = min(S, u)
    info = comm.all_gather_ints([D, s])
    dims = [d for d, _ in info]
    if any(d != D for d in dims):
        raise MeshError(f"all shards must share dim, got {dims}")
    pad = uniq.new_zeros((S, D))
    if s:
        pos = (torch.arange(s, dtype=torch.int64) * u) // s
        pad[:s] = uniq[pos.to(uniq.device)]
    every_pad = comm.all_gather_fixed(pad)
    every = torch.cat([every_pad[g * S:g * S + info[g][1]] for g in range(G)])
    m_all = every.shape[0]
    if m_all:
        ident = torch.arange(m_all, dtype=torch.int32, device=every.device).view(m_all, 1)
        sorted_samples, _ = backend.reindex(every, ident)
        m = sorted_samples.shape[0]
        pick = (torch.arange(1, G, dtype=torch.int64) * m) // G
        splitters = sorted_samples[pick.to(sorted_samples.device)]
    else:
        splitters = uniq.new_empty((0, D))
    # 3. partition the sorted keys into G contiguous ranges (bounds stay on the device) and exchange
    lb = backend.lower_bound(uniq, splitters) if splitters.shape[0] else None
    if isinstance(lb, torch.Tensor):
        bounds = torch.cat([torch.zeros(1, dtype=torch.int64, device=lb.device), lb,
                            torch.full((1,), u, dtype=torch.int64, device=lb.device)])
        send_dev = bounds[1:] - bounds[:-1]
    else:  # host backends (tests)
        b = [0] + (list(lb) if lb is not None else [u] * (G - 1)) + [u]
        bounds = None
        send_dev = torch.tensor([b[g + 1] - b[g] for g in range(G)], dtype=torch.int64)
    C = comm.count_matrix(send_dev)
    send_counts = C[me]
    mark("split")
    recv_keys, recv_counts = comm.all_to_all(uniq, send_counts, C, bounds)
    mark("exchange")
    # 4. merge what arrived (G sorted, duplicate-free runs): sorted unique keys of this range +
    #    the rank of each received key
    n_recv = recv_keys.shape[0]
    # merging beats re-sorting the runs (tools/merge_runs_bench.py: 8 runs / 106M rows 5.2 vs 6.9 ms,
    # 4 runs / 29M rows 1.2 vs 2.2 ms, 16 runs / 194M rows 11.7 vs 12.0 ms)
    if n_recv and hasattr(backend, "merge_unique") and D <= 8:
        mine_buf, rank_of, cnt = backend.merge_unique(recv_keys, recv_counts)
        sizes = [v[0] for v in comm.all_gather_ints_dev(cnt)] if hasattr(comm, "all_gather_ints_dev") \
            else comm.all_gather_int(int(cnt.item()))
        mine = mine_buf[:sizes[me]]
    else:
        if n_recv:
            ident = torch.arange(n_recv, dtype=torch.int32, device=recv_keys.device).view(n_recv, 1)
            mine, rank_of = backend.reindex(recv_keys, ident)
        else:
            mine, rank_of = recv_keys.new_empty((0, D)), recv_keys.new_empty((0, 1))
        sizes = comm.all_gather_int(mine.shape[0])
    mark("merge")
    # 5. global offsets
    offset = sum(sizes[:me])
    total = sum(sizes)
    if total >= 1 << 32:
        raise MeshError(f"global unique count {total} exceeds 32-bit index range")
    gid = (rank_of.reshape(-1).to(torch.int64) + offset).to(torch.int32)
    # 6. reverse exchange: global id of every local unique key, in local order (the counts are the
    #    transposed forward counts: no second count exchange)
    CT = [[C[g][s] for g in range(G)] for s in range(G)]
    new_of_local, _ = comm.all_to_all(gid, recv_counts, CT)
    mark("reverse")
    # 7. remap this rank's elements
    status = torch.zeros(1, dtype=torch.int32, device=local_out.device) if check else None
    if status is not None and hasattr(backend, "merge_unique"):
        out = backend.gather(new_of_local, local_out.reshape(-1), status).view(local_out.shape)
        if int(status.item()):
            raise MeshError("remap table index out of range (internal)")
    else:
        out = backend.gather(new_of_local, local_out.reshape(-1)).view(local_out.shape)
    mark("remap")
    if cuda:
        torch.cuda.current_stream(vertex_bits.device).synchronize()
        names = list(ev)
        for a, b in zip(names, names[1:]):
            timing[f"{b}_ms"] = ev[a].elapsed_time(ev[b])
        row = 4 * D
        timing["exchange_bytes_out"] = (u - send_counts[me]) * row + (n_recv - recv_counts[me]) * 4
        timing["exchange_bytes_in"] = (n_recv - recv_counts[me]) * row + (u - send_counts[me]) * 4
    return DistResult(mine, offset, total, out)


def run_threads(shards, backend_factory, samples_per_rank: int = 1024) -> list[DistResult]:
    """Run reindex_distributed over G in-process ranks (one thread each)."""
    G = len(shards)
    hub = ThreadHub(G)
    results: list = [None] * G
    errors: list = []

    def body(r):
        try:
            v, e = shards[r]
            results[r] = reindex_distributed(v, e, ThreadComm(hub, r), backend_factory(r), samples_per_rank)
        except BaseException as exc:  # noqa: BLE001 - surfaced below
            errors.append(exc)
            hub.barrier.abort()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return results


__all__ = ["Comm", "TorchComm", "SymmComm", "ThreadComm", "ThreadHub", "CudaBackend", "DistResult",
           "reindex_distributed", "run_threads"]
