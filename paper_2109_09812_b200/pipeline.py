"""Drop-in ``reindex``: the reference operator API over the CUDA C-ABI.

Reference interface (``pkg/src/remeshx/pipeline.py:133-157``)::

    reindex(mesh: Mesh) -> tuple[Mesh, ReindexScratch]

Same argument meaning, same result types and the same errors:

* out-of-range indices    -> ``InvalidMeshError`` with the reference's ``Issue``
  list (``mesh.py:103-105``; detected on the GPU by K1, listed on the cold path);
* zero elements           -> ``Mesh.empty(dim, arity)`` and an all-false
  ``is_used`` (``pipeline.py:142-146``);
* ``n_vertices >= 2**32`` -> ``MeshError`` (``mesh.py:59-60``).

Three entry levels share one native call (``rmx_reindex``):

* :func:`reindex`         -- numpy in, numpy out (the reference signature);
* :class:`Reindexer`      -- fixed-capacity device + pinned host buffers for
  repeated host-to-host calls (the end-to-end path bench.py times);
* :func:`reindex_tensors` -- device-resident torch tensors in and out.

PyTorch is only the buffer/stream plumbing; all arithmetic is in the CUDA
library.  There is no CPU fallback: a missing library raises.
"""
from __future__ import annotations

import ctypes
import threading
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, hostio
from .mesh import InvalidMeshError, Mesh, MeshError, validate

_SCRATCH_FIELDS = ("is_used", "org_id", "nodup", "new_idx", "perm")


def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2109_09812_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def workspace_bytes(n_vertices: int, dim: int, n_elements: int = 0, arity: int = 1) -> int:
    return int(_native.lib().rmx_workspace_bytes(n_vertices, dim, n_elements, arity))


def _raise_for(rc: int) -> None:
    if rc == _native.RMX_OK:
        return
    msg = _native.lib().rmx_strerror(rc).decode()
    if rc in (_native.RMX_EINVAL, _native.RMX_ERANGE):
        raise MeshError(msg)
    raise RuntimeError(f"CUDA re-indexing failed ({rc}): {msg}")


def host_tensor(a: np.ndarray) -> torch.Tensor:
    """Zero-copy torch view of a host array that is only read (copied to the device).

    Mesh arrays are read-only; torch warns on wrapping them although nothing writes.
    """
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(a)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


@dataclass
class DeviceResult:
    """Device-resident result of :func:`reindex_tensors`.

    ``vertices`` is an int32 ``(U, dim)`` bit view, ``elements`` int32
    ``(E, arity)``; ``scratch`` maps the ReindexScratch field names to device
    tensors when requested.
    """

    vertices: torch.Tensor
    elements: torch.Tensor
    new_count: int
    scratch: dict | None


def launch(vtx: torch.Tensor, n_vertices: int, dim: int, idx: torch.Tensor, n_elements: int, arity: int,
           out_vtx: torch.Tensor, out_idx: torch.Tensor, info: torch.Tensor, workspace: torch.Tensor,
           scratch: dict | None = None, stream: torch.cuda.Stream | None = None, events=None) -> None:
    """Enqueue the pipeline on ``stream`` (no synchronisation).

    ``info`` is an int64 device tensor of 2 elements: [0] receives the output
    vertex count, the low word of [1] the status bits.  ``events`` is an
    optional sequence of raw cudaEvent_t handles recorded at stage boundaries.
    """
    lib = _native.lib()
    sc = None
    if scratch is not None:
        sc = _native.Scratch(*[_ptr(scratch.get(f)) for f in _SCRATCH_FIELDS])
    s = (stream or torch.cuda.current_stream(vtx.device if vtx is not None else idx.device)).cuda_stream
    base = info.data_ptr()
    args = (_ptr(vtx), n_vertices, dim, _ptr(idx), n_elements, arity, _ptr(out_vtx), _ptr(out_idx),
            base, base + 8, workspace.data_ptr() if workspace is not None else None,
            workspace.numel() if workspace is not None else 0,
            ctypes.byref(sc) if sc is not None else None, s)
    if events:
        arr = (ctypes.c_void_p * len(events))(*events)
        rc = lib.rmx_reindex_profiled(*args, arr, len(events))
    else:
        rc = lib.rmx_reindex(*args)
    _raise_for(rc)


class PipelineGraph:
    """``rmx_reindex`` for fixed buffers and sizes captured once as a CUDA graph.

    Sections a given input does not need (AoS rows vs packed keys, each sort
    pass) are conditional nodes the plan kernel switches on the device, so
    a launch runs only the kernels that do work, and the whole pipeline is one
    host call (for embedding in a caller's graph, or host-bound loops).  The
    tensors are kept alive by the object; results land in ``out_vtx`` /
    ``out_idx`` / ``info`` like :func:`launch`.  Measured on B200 the device
    time equals direct launches within a few percent (C2 8.87 vs 8.94 ms): a
    skipped conditional node costs about what a no-op kernel did.
    """

    def __init__(self, vtx, n_vertices, dim, idx, n_elements, arity, out_vtx, out_idx, info, workspace):
        lib = _native.lib()
        self._keep = (vtx, idx, out_vtx, out_idx, info, workspace)
        base = info.data_ptr()
        h = ctypes.c_void_p()
        rc = lib.rmx_graph_create(_ptr(vtx), n_vertices, dim, _ptr(idx), n_elements, arity, _ptr(out_vtx),
                                  _ptr(out_idx), base, base + 8, workspace.data_ptr(), workspace.numel(), None,
                                  ctypes.byref(h))
        _raise_for(rc)
        self._h = h

    def launch(self, stream: torch.cuda.Stream) -> None:
        _raise_for(_native.lib().rmx_graph_launch(self._h, stream.cuda_stream))

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _native.lib().rmx_graph_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the module globals may be gone
            pass


def _alloc_scratch(n_vertices: int, device) -> dict:
    return dict(is_used=torch.empty(n_vertices, dtype=torch.uint8, device=device),
                org_id=torch.empty(n_vertices, dtype=torch.int32, device=device),
                nodup=torch.empty(n_vertices, dtype=torch.uint8, device=device),
                new_idx=torch.empty(n_vertices, dtype=torch.int32, device=device),
                perm=torch.empty(n_vertices, dtype=torch.int32, device=device))


def reindex_tensors(vertex_bits: torch.Tensor, elements: torch.Tensor, *, scratch: bool = False,
                    stream: torch.cuda.Stream | None = None) -> DeviceResult:
    """Re-index device-resident data: ``vertex_bits`` (V, D) int32/uint32 words,
    ``elements`` (E, K) int32/uint32 indices, both contiguous on one CUDA device.

    Synchronises once to learn the output size.  Raises InvalidMeshError (with
    issues found on the device) for out-of-range indices.
    """
    if vertex_bits.dim() != 2 or elements.dim() != 2:
        raise MeshError("vertex_bits must be (V, D) and elements (E, K)")
    if vertex_bits.element_size() != 4 or elements.element_size() != 4:
        raise MeshError("vertex_bits and elements must hold 32-bit words")
    vertex_bits = vertex_bits.contiguous()
    elements = elements.contiguous()
    dev = vertex_bits.device
    V, D = vertex_bits.shape
    E, K = elements.shape
    if V >= 1 << 32:
        raise MeshError(f"vertex count {V} exceeds 32-bit index range")
    out_v = torch.empty((V, D), dtype=torch.int32, device=dev)
    out_e = torch.empty((E, K), dtype=torch.int32, device=dev)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(max(workspace_bytes(V, D, E, K), 1) if E else 1, dtype=torch.uint8, device=dev)
    sc = _alloc_scratch(V, dev) if scratch else None
    launch(vertex_bits, V, D, elements, E, K, out_v, out_e, info, ws, sc, stream)
    count, status = (int(x) for x in info.cpu())
    if status & _native.RMX_STATUS_INDEX_OUT_OF_RANGE:
        bad = torch.nonzero(elements.to(torch.int64) & 0xFFFFFFFF >= V).cpu().numpy()
        host = elements.cpu().numpy().view(np.uint32)
        from .mesh import Issue
        raise InvalidMeshError([Issue(int(e), int(s), int(host[e, s])) for e, s in bad])
    if E == 0:
        out_v = out_v[:0]
    else:
        out_v = out_v[:count]
    return DeviceResult(out_v, out_e, count, sc)


def reindex_tensors_lean(vertex_bits: torch.Tensor, elements: torch.Tensor, *,
                         stream: torch.cuda.Stream | None = None) -> DeviceResult:
    """Memory-lean device re-index (opt-in, tensor API only).

    ``vertex_bits`` is OVERWRITTEN: once the sort keys are built it serves as the
    second sort buffer, so the workspace is ~40 B per vertex instead of ~52 and
    no output-vertex buffer of V rows is needed (C5, 3.15B vertex slots, fits
    one 180 GB B200).  The returned vertices are a view of the workspace or of
    ``vertex_bits``.  Needs keys that pack into 64 bits (lattice-like or
    quantised data: MeshError otherwise), dim >= 3, an even vertex count; small
    meshes take :func:`reindex_tensors`.  Not a drop-in for the reference
    (which never mutates its input, pipeline.py:133-157).
    """
    lib = _native.lib()
    if vertex_bits.dim() != 2 or elements.dim() != 2 or vertex_bits.element_size() != 4 \
            or elements.element_size() != 4:
        raise MeshError("vertex_bits must be (V, D) and elements (E, K) of 32-bit words")
    if not vertex_bits.is_contiguous():
        raise MeshError("lean mode works in place: vertex_bits must be contiguous")
    V, D = vertex_bits.shape
    E, K = elements.shape
    if E == 0 or D < 3 or V % 2 or V <= 8192:
        return reindex_tensors(vertex_bits, elements, stream=stream)
    if V >= 1 << 32:
        raise MeshError(f"vertex count {V} exceeds 32-bit index range")
    dev = vertex_bits.device
    elements = elements.contiguous()
    ws = torch.empty(int(lib.rmx_lean_workspace_bytes(V, D, E, K)), dtype=torch.uint8, device=dev)
    out_e = torch.empty((E, K), dtype=torch.int32, device=dev)
    info = torch.zeros(3, dtype=torch.int64, device=dev)  # count, status, where
    s = (stream or torch.cuda.current_stream(dev)).cuda_stream
    base = info.data_ptr()
    _raise_for(lib.rmx_reindex_lean(vertex_bits.data_ptr(), V, D, elements.data_ptr(), E, K, out_e.data_ptr(), base,
                                    base + 8, base + 16, ws.data_ptr(), ws.numel(), s))
    count, status, where = (int(x) for x in info.cpu())
    if status & _native.RMX_STATUS_INDEX_OUT_OF_RANGE:
        bad = torch.nonzero(elements.to(torch.int64) & 0xFFFFFFFF >= V).cpu().numpy()
        host = elements.cpu().numpy().view(np.uint32)
        from .mesh import Issue
        raise InvalidMeshError([Issue(int(e), int(s_), int(host[e, s_])) for e, s_ in bad])
    if status & _native.RMX_STATUS_LEAN_UNSUPPORTED:
        raise MeshError("lean mode needs keys that pack into 64 bits; this vertex set varies in more "
                        "(use reindex_tensors)")
    if where == 0:
        off = int(lib.rmx_lean_result_offset(V, D))
        verts = ws[off:off + count * D * 4].view(torch.int32).view(count, D)
    else:
        verts = vertex_bits.view(-1)[:count * D].view(count, D)
    return DeviceResult(verts, out_e, count, None)


class ReindexScratch:
    """Intermediates of one run (reference ``ReindexScratch``, pipeline.py:24-38).

    ``new_count`` is known immediately.  The array fields are materialised on
    first access by re-running the (deterministic) device pipeline with
    scratch outputs enabled, so the hot path never pays for them.
    """

    __slots__ = ("_src", "_count", "_arrays", "_device")

    def __init__(self, vertices: np.ndarray, elements: np.ndarray, new_count: int, device):
        object.__setattr__(self, "_src", (vertices, elements))
        object.__setattr__(self, "_count", int(new_count))
        object.__setattr__(self, "_arrays", None)
        object.__setattr__(self, "_device", device)

    def __setattr__(self, name, value):
        raise AttributeError("ReindexScratch is immutable")

    @property
    def new_count(self) -> int:
        return self._count

    def _materialise(self) -> dict:
        if self._arrays is None:
            vertices, elements = self._src
            V, D = vertices.shape
            E, K = elements.shape
            dev = self._device
            with torch.cuda.device(dev):
                vtx_d = torch.empty((V, D), dtype=torch.int32, device=dev)
                idx_d = torch.empty((E, K), dtype=torch.int32, device=dev)
                hostio.to_device(np.ascontiguousarray(vertices), vtx_d)
                hostio.to_device(np.ascontiguousarray(elements), idx_d)
                res = reindex_tensors(vtx_d, idx_d, scratch=True)
                sc = res.scratch
                n = V if E else 0
                arrays = dict(
                    is_used=hostio.to_host(sc["is_used"]).view(bool),
                    org_id=hostio.to_host(sc["org_id"][:n]).view(np.uint32),
                    nodup=hostio.to_host(sc["nodup"][:n]).view(bool),
                    new_idx=hostio.to_host(sc["new_idx"][:n]).view(np.uint32),
                    perm=hostio.to_host(sc["perm"][:n]).view(np.uint32))
            for a in arrays.values():
                a.flags.writeable = False
            object.__setattr__(self, "_arrays", arrays)
        return self._arrays

    @property
    def is_used(self) -> np.ndarray:
        return self._materialise()["is_used"]

    @property
    def org_id(self) -> np.ndarray:
        return self._materialise()["org_id"]

    @property
    def nodup(self) -> np.ndarray:
        return self._materialise()["nodup"]

    @property
    def new_idx(self) -> np.ndarray:
        return self._materialise()["new_idx"]

    @property
    def perm(self) -> np.ndarray:
        return self._materialise()["perm"]

    def __repr__(self):
        return f"ReindexScratch(new_count={self._count})"


def _host_arrays(mesh) -> tuple[np.ndarray, np.ndarray]:
    """float32/uint32 C-contiguous arrays of a Mesh (or any .vertices/.elements object)."""
    if isinstance(mesh, Mesh):
        return mesh.vertices, mesh.elements
    v = np.ascontiguousarray(mesh.vertices, dtype=np.float32)
    e = np.ascontiguousarray(mesh.elements, dtype=np.uint32)
    if v.ndim != 2 or v.shape[1] < 1 or e.ndim != 2 or e.shape[1] < 1:
        raise MeshError(f"bad mesh shapes {v.shape} / {e.shape}")
    if v.shape[0] >= 1 << 32:
        raise MeshError(f"vertex count {v.shape[0]} exceeds 32-bit index range")
    if v.flags.writeable or e.flags.writeable:     # snapshot for the lazy scratch
        v, e = v.copy(), e.copy()
        v.flags.writeable = False
        e.flags.writeable = False
    return v, e


def reindex(mesh, device=None) -> tuple[Mesh, ReindexScratch]:
    """Remove duplicate and unused vertices (reference pipeline.py:133-157).

    Output vertices are the bitwise-sorted unique used rows; element indices
    are remapped accordingly; the soup is preserved bit for bit.
    """
    vertices, elements = _host_arrays(mesh)
    dev = _device(device)
    V, D = vertices.shape
    E, K = elements.shape
    if E == 0:
        return Mesh.empty(dim=D, arity=K), ReindexScratch(vertices, elements, 0, dev)
    if vertices.nbytes + elements.nbytes <= SMALL_CALL_BYTES:
        return _reindex_small(vertices, elements, dev)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        vtx_d = torch.empty((V, D), dtype=torch.int32, device=dev)
        idx_d = torch.empty((E, K), dtype=torch.int32, device=dev)
        hostio.to_device(vertices, vtx_d)
        hostio.to_device(elements, idx_d)
        out_v = torch.empty((V, D), dtype=torch.int32, device=dev)
        out_e = torch.empty((E, K), dtype=torch.int32, device=dev)
        info = torch.zeros(2, dtype=torch.int64, device=dev)
        ws = torch.empty(workspace_bytes(V, D, E, K), dtype=torch.uint8, device=dev)
        launch(vtx_d, V, D, idx_d, E, K, out_v, out_e, info, ws, None, stream)
        del vtx_d, idx_d, ws
        if _pinned_results():
            # results land in pinned blocks of torch's caching host allocator (reused once the
            # caller drops an earlier result): one DMA per array, no staging copy, no page faults
            # in fresh numpy pages; the element copy starts before the count is known
            host_info = torch.empty(2, dtype=torch.int64, pin_memory=True)
            host_e_t = torch.empty((E, K), dtype=torch.int32, pin_memory=True)
            host_info.copy_(info, non_blocking=True)
            host_e_t.copy_(out_e, non_blocking=True)
            stream.synchronize()
            count, status = (int(x) for x in host_info)
            if status & _native.RMX_STATUS_INDEX_OUT_OF_RANGE:
                raise InvalidMeshError(validate(_Arrays(vertices, elements)))
            host_v_t = torch.empty((count, D), dtype=torch.int32, pin_memory=True)
            if count:
                host_v_t.copy_(out_v[:count], non_blocking=True)
                stream.synchronize()
            host_v = host_v_t.numpy().view(np.float32)
            host_e = host_e_t.numpy().view(np.uint32)
        else:
            count, status = (int(x) for x in info.cpu())
            if status & _native.RMX_STATUS_INDEX_OUT_OF_RANGE:
                raise InvalidMeshError(validate(_Arrays(vertices, elements)))
            host_v = hostio.to_host(out_v[:count]).view(np.float32)
            host_e = hostio.to_host(out_e).view(np.uint32)
    return Mesh._adopt(host_v, host_e), ReindexScratch(vertices, elements, count, dev)


def _pinned_results() -> bool:
    """RMX_PINNED_RESULTS=0: return results in ordinary pageable numpy arrays (staged copies)."""
    import os
    return os.environ.get("RMX_PINNED_RESULTS", "1") != "0"


# Meshes up to this many input bytes take one staged round trip: one pinned
# buffer up, one launch, one pinned buffer down, one synchronisation.
SMALL_CALL_BYTES = 4 << 20


class _SmallBuffers(threading.local):
    """Per-thread, per-device device + pinned host buffers of the small-call path (grown on demand)."""

    def __init__(self):
        self.by_dev = {}

    def get(self, dev: torch.device, nbytes: int):
        cur = self.by_dev.get(dev)
        if cur is None or cur[0].numel() < nbytes:
            cap = max(nbytes, 1 << 20)
            cur = (torch.empty(cap, dtype=torch.uint8, device=dev),
                   torch.empty(cap, dtype=torch.uint8, pin_memory=True))
            self.by_dev[dev] = cur
        return cur


_small = _SmallBuffers()


def _reindex_small(vertices: np.ndarray, elements: np.ndarray, dev: torch.device):
    """reindex() for small meshes: [vertices | elements] up in one copy, [info | out vertices |
    out elements] down in one copy, one stream synchronisation."""
    V, D = vertices.shape
    E, K = elements.shape
    nv, ne = vertices.nbytes, elements.nbytes

    def al(x):
        return (x + 255) & ~255

    o_idx = al(nv)
    o_info = al(o_idx + ne)
    o_ov = o_info + 16
    o_oe = al(o_ov + nv)
    o_ws = al(o_oe + ne)
    wsb = workspace_bytes(V, D, E, K)
    with torch.cuda.device(dev):
        dbuf, hbuf = _small.get(dev, o_ws + wsb)
        h = hbuf.numpy()
        h[:nv] = vertices.reshape(-1).view(np.uint8)
        h[o_idx:o_idx + ne] = elements.reshape(-1).view(np.uint8)
        stream = torch.cuda.current_stream(dev)
        dbuf[:o_idx + ne].copy_(hbuf[:o_idx + ne], non_blocking=True)
        base = dbuf.data_ptr()
        lib = _native.lib()
        _raise_for(lib.rmx_reindex(base, V, D, base + o_idx, E, K, base + o_ov, base + o_oe, base + o_info,
                                   base + o_info + 8, base + o_ws, wsb, None, stream.cuda_stream))
        hbuf[o_info:o_oe + ne].copy_(dbuf[o_info:o_oe + ne], non_blocking=True)
        stream.synchronize()
        count, status = (int(x) for x in h[o_info:o_info + 16].view(np.int64))
        if status & _native.RMX_STATUS_INDEX_OUT_OF_RANGE:
            raise InvalidMeshError(validate(_Arrays(vertices, elements)))
        host_v = h[o_ov:o_ov + count * D * 4].view(np.float32).reshape(count, D).copy()
        host_e = h[o_oe:o_oe + ne].view(np.uint32).reshape(E, K).copy()
    return Mesh._adopt(host_v, host_e), ReindexScratch(vertices, elements, count, dev)


class _Arrays:
    __slots__ = ("vertices", "elements")

    def __init__(self, vertices, elements):
        self.vertices = vertices
        self.elements = elements


class Reindexer:
    """Fixed-capacity buffers for repeated host-to-host re-indexing.

    ``run(vertices_pinned, elements_pinned)`` copies the inputs host->device,
    runs the pipeline, and copies the result back into pinned host buffers;
    returns numpy views ``(vertices (U, D) float32, elements (E, K) uint32)``
    valid until the next call.  Inputs should be pinned torch tensors (see
    :meth:`pinned_inputs`) so the copies run at full PCIe speed.
    """

    def __init__(self, n_vertices: int, dim: int, n_elements: int, arity: int, device=None):
        self.device = _device(device)
        self.V, self.D, self.E, self.K = int(n_vertices), int(dim), int(n_elements), int(arity)
        dev = self.device
        self.vtx_d = torch.empty((self.V, self.D), dtype=torch.int32, device=dev)
        self.idx_d = torch.empty((self.E, self.K), dtype=torch.int32, device=dev)
        self.out_v = torch.empty((self.V, self.D), dtype=torch.int32, device=dev)
        self.out_e = torch.empty((self.E, self.K), dtype=torch.int32, device=dev)
        self.info = torch.zeros(2, dtype=torch.int64, device=dev)
        self.ws = torch.empty(max(1, workspace_bytes(self.V, self.D, self.E, self.K)), dtype=torch.uint8,
                              device=dev)
        self.host_v = torch.empty((self.V, self.D), dtype=torch.int32, pin_memory=True)
        self.host_e = torch.empty((self.E, self.K), dtype=torch.int32, pin_memory=True)
        self.host_info = torch.empty(2, dtype=torch.int64, pin_memory=True)
        self.stream = torch.cuda.Stream(dev)

    def pinned_inputs(self, vertices: np.ndarray, elements: np.ndarray) -> tuple[torch.Tensor, torch.Tensor]:
        v = torch.empty((self.V, self.D), dtype=torch.int32, pin_memory=True)
        e = torch.empty((self.E, self.K), dtype=torch.int32, pin_memory=True)
        v.numpy()[:] = np.ascontiguousarray(vertices, dtype=np.float32).view(np.int32)
        e.numpy()[:] = np.ascontiguousarray(elements, dtype=np.uint32).view(np.int32)
        return v, e

    def bytes_per_call(self, count: int) -> tuple[int, int]:
        h2d = self.V * self.D * 4 + self.E * self.K * 4
        d2h = 16 + count * self.D * 4 + self.E * self.K * 4
        return h2d, d2h

    def run(self, vertices_pinned: torch.Tensor, elements_pinned: torch.Tensor):
        s = self.stream
        with torch.cuda.device(self.device), torch.cuda.stream(s):
            self.vtx_d.copy_(vertices_pinned, non_blocking=True)
            self.idx_d.copy_(elements_pinned, non_blocking=True)
            launch(self.vtx_d, self.V, self.D, self.idx_d, self.E, self.K, self.out_v, self.out_e,
                   self.info, self.ws, None, s)
            self.host_info.copy_(self.info, non_blocking=True)
            # the element result size is known up front: start it before the count arrives
            self.host_e.copy_(self.out_e, non_blocking=True)
            s.synchronize()
            count, status = (int(x) for x in self.host_info)
            if status & _native.RMX_STATUS_INDEX_OUT_OF_RANGE:
                host_v = vertices_pinned.numpy().view(np.float32)
                host_e = elements_pinned.numpy().view(np.uint32)
                raise InvalidMeshError(validate(_Arrays(host_v, host_e)))
            if count:
                self.host_v[:count].copy_(self.out_v[:count], non_blocking=True)
            s.synchronize()
        self.last_count = count
        return (self.host_v[:count].numpy().view(np.float32), self.host_e.numpy().view(np.uint32))


class _Slot:
    """Device + pinned host buffers of one in-flight mesh of a :class:`ReindexStream`."""

    def __init__(self, V: int, D: int, E: int, K: int, dev: torch.device):
        self.vtx_d = torch.empty((V, D), dtype=torch.int32, device=dev)
        self.idx_d = torch.empty((E, K), dtype=torch.int32, device=dev)
        self.out_v = torch.empty((V, D), dtype=torch.int32, device=dev)
        self.out_e = torch.empty((E, K), dtype=torch.int32, device=dev)
        self.info = torch.zeros(2, dtype=torch.int64, device=dev)
        self.host_v = torch.empty((V, D), dtype=torch.int32, pin_memory=True)
        self.host_e = torch.empty((E, K), dtype=torch.int32, pin_memory=True)
        self.host_info = torch.empty(2, dtype=torch.int64, pin_memory=True)
        self.h2d_done = torch.cuda.Event()
        self.comp_done = torch.cuda.Event()
        self.d2h_done = torch.cuda.Event()
        self.used = False
        self.inputs = None
        self.shape = (0, 0)


class ReindexStream:
    """Pipelined host-to-host re-indexing of a sequence of meshes.

    The three engines of the GPU work on different meshes at once: while mesh
    k is re-indexed on the compute stream, mesh k+1's vertices and elements
    cross PCIe host->device on one copy stream and mesh k-1's result comes
    back device->host on the other (the link is full duplex).  The kernels
    share one workspace (compute is serialised on one stream); inputs and
    results are double-buffered.

    ``run(batches)`` takes an iterable of pinned ``(vertices int32 (V, D),
    elements int32 (E, K))`` tensors with V, E within the capacity given at
    construction and yields ``(vertices (U, D) float32, elements (E, K)
    uint32)`` numpy views in input order.  A yielded result stays valid until
    the generator is advanced again (copy it to keep it).  An out-of-range
    index raises :class:`InvalidMeshError` for that mesh, like :func:`reindex`.
    """

    def __init__(self, max_vertices: int, dim: int, max_elements: int, arity: int, device=None, depth: int = 2):
        self.device = _device(device)
        self.V, self.D, self.E, self.K = int(max_vertices), int(dim), int(max_elements), int(arity)
        if depth < 2:
            raise ValueError("depth must be >= 2")
        dev = self.device
        with torch.cuda.device(dev):
            self.slots = [_Slot(self.V, self.D, self.E, self.K, dev) for _ in range(depth)]
            self.ws = torch.empty(max(1, workspace_bytes(self.V, self.D, self.E, self.K)), dtype=torch.uint8,
                                  device=dev)
            self.h2d = torch.cuda.Stream(dev)
            self.comp = torch.cuda.Stream(dev)
            self.d2h = torch.cuda.Stream(dev)
        self.last_counts: list[int] = []

    def bytes_per_mesh(self, n_vertices: int, n_elements: int, count: int) -> tuple[int, int]:
        h2d = n_vertices * self.D * 4 + n_elements * self.K * 4
        d2h = 16 + count * self.D * 4 + n_elements * self.K * 4
        return h2d, d2h

    def _submit(self, slot: _Slot, vertices: torch.Tensor, elements: torch.Tensor) -> None:
        V, E = vertices.shape[0], elements.shape[0]
        if vertices.shape[1:] != (self.D,) or elements.shape[1:] != (self.K,):
            raise MeshError(f"mesh shapes {tuple(vertices.shape)} / {tuple(elements.shape)} do not match "
                            f"dim={self.D} arity={self.K}")
        if V > self.V or E > self.E:
            raise MeshError(f"mesh ({V} vertices, {E} elements) exceeds the stream capacity ({self.V}, {self.E})")
        if slot.used:  # the previous mesh of this slot must be off its buffers
            self.h2d.wait_event(slot.comp_done)
        with torch.cuda.stream(self.h2d):
            slot.vtx_d[:V].copy_(vertices, non_blocking=True)
            slot.idx_d[:E].copy_(elements, non_blocking=True)
            slot.h2d_done.record(self.h2d)
        self.comp.wait_event(slot.h2d_done)
        if slot.used:
            self.comp.wait_event(slot.d2h_done)
        with torch.cuda.stream(self.comp):
            if E:
                launch(slot.vtx_d, V, self.D, slot.idx_d, E, self.K, slot.out_v, slot.out_e, slot.info, self.ws,
                       None, self.comp)
            else:
                slot.info.zero_()
            slot.host_info.copy_(slot.info, non_blocking=True)
            slot.comp_done.record(self.comp)
        slot.used = True
        slot.inputs = (vertices, elements)
        slot.shape = (V, E)

    def _finish(self, slot: _Slot):
        V, E = slot.shape
        # the element result has a known size: start it before the host learns the count.
        # (Enqueued here, not at submit: the copy stream must not queue behind the next mesh.)
        self.d2h.wait_event(slot.comp_done)
        with torch.cuda.stream(self.d2h):
            if E:
                slot.host_e[:E].copy_(slot.out_e[:E], non_blocking=True)
        slot.comp_done.synchronize()
        count, status = (int(x) for x in slot.host_info)
        if status & _native.RMX_STATUS_INDEX_OUT_OF_RANGE:
            self.synchronize()
            hv, he = slot.inputs
            raise InvalidMeshError(validate(_Arrays(hv.numpy().view(np.float32), he.numpy().view(np.uint32))))
        with torch.cuda.stream(self.d2h):
            if count:
                slot.host_v[:count].copy_(slot.out_v[:count], non_blocking=True)
            slot.d2h_done.record(self.d2h)
        slot.d2h_done.synchronize()
        slot.inputs = None
        self.last_counts.append(count)
        return (slot.host_v[:count].numpy().view(np.float32), slot.host_e[:E].numpy().view(np.uint32))

    def run(self, batches):
        depth = len(self.slots)
        pending: list[_Slot] = []
        k = 0
        with torch.cuda.device(self.device):
            for vertices, elements in batches:
                slot = self.slots[k % depth]
                self._submit(slot, vertices, elements)
                pending.append(slot)
                k += 1
                if len(pending) == depth:
                    yield self._finish(pending.pop(0))
            while pending:
                yield self._finish(pending.pop(0))

    def synchronize(self) -> None:
        for s in (self.h2d, self.comp, self.d2h):
            s.synchronize()
