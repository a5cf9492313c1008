"""RMX1 binary container, read straight into pinned host and device memory.

Format (reference ``pkg/src/remeshx/fileio.py:1-12,125-156``), little-endian:
28-byte header ``<4sIIQQ`` = magic ``RMX1``, u32 dim, u32 arity, u64 vertex
count, u64 element count; then dim x f32 per vertex, then arity x u32 per
element.  Same validation and errors as the reference ``read_bin``
(``FormatError`` for a short header, bad magic, dim/arity < 1, truncated
payload, trailing bytes).

* :func:`read_bin` / :func:`write_bin` -- host Mesh in / out (bit-exact round
  trip, like the reference);
* :func:`load_bin_tensors` -- the payload is read with ``readinto`` into two
  pinned staging buffers in turn while the previous chunk is copied
  host->device on a copy stream: the file lands in HBM with one pass over the
  bytes and the disk read overlapping PCIe;
* :func:`reindex_file` -- RMX1 in -> device re-index -> RMX1 out.
"""
from __future__ import annotations

import os
import struct

import numpy as np
import torch

from .mesh import Mesh, MeshError, require_valid
from .pipeline import _device

MAGIC = b"RMX1"
HEADER = struct.Struct("<4sIIQQ")
CHUNK = 64 << 20


class FormatError(MeshError):
    """Malformed or truncated mesh file (reference fileio.py:24-25)."""


def _read_header(handle, path) -> tuple[int, int, int, int]:
    header = handle.read(HEADER.size)
    if len(header) < HEADER.size:
        raise FormatError(f"{path}: truncated header ({len(header)} bytes)")
    magic, dim, arity, n_vertices, n_elements = HEADER.unpack(header)
    if magic != MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    if dim < 1 or arity < 1:
        raise FormatError(f"{path}: invalid dim={dim} arity={arity}")
    return dim, arity, n_vertices, n_elements


def _check_payload(handle, path, want: int) -> None:
    have = os.fstat(handle.fileno()).st_size - HEADER.size
    if have < want:
        raise FormatError(f"{path}: truncated payload")
    if have > want:
        raise FormatError(f"{path}: trailing bytes after payload")


def _bytes(a: np.ndarray) -> memoryview:
    """Flat writable/readable byte view of a C-contiguous array (empty arrays too)."""
    return memoryview(a.reshape(-1).view(np.uint8))


def _readinto_exact(handle, view: memoryview, path) -> None:
    got = 0
    while got < len(view):
        n = handle.readinto(view[got:])
        if not n:
            raise FormatError(f"{path}: truncated payload")
        got += n


def write_bin(mesh, path) -> None:
    """Write the RMX1 container (reference fileio.py:125-133)."""
    require_valid(mesh)
    v = np.ascontiguousarray(mesh.vertices, dtype="<f4")
    e = np.ascontiguousarray(mesh.elements, dtype="<u4")
    with open(path, "wb") as handle:
        handle.write(HEADER.pack(MAGIC, v.shape[1], e.shape[1], v.shape[0], e.shape[0]))
        handle.write(_bytes(v))
        handle.write(_bytes(e))


def read_bin(path) -> Mesh:
    """Read the RMX1 container into a host Mesh (reference fileio.py:136-156)."""
    with open(path, "rb") as handle:
        dim, arity, nv, ne = _read_header(handle, path)
        _check_payload(handle, path, dim * 4 * nv + arity * 4 * ne)
        v = np.empty((nv, dim), np.float32)
        e = np.empty((ne, arity), np.uint32)
        _readinto_exact(handle, _bytes(v), path)
        _readinto_exact(handle, _bytes(e), path)
    return Mesh._adopt(v, e)


def load_bin_tensors(path, device=None, chunk: int = CHUNK) -> tuple[torch.Tensor, torch.Tensor]:
    """RMX1 file -> (vertex bits int32 (V, D), elements int32 (E, K)) on the device.

    The payload is streamed through two pinned staging buffers: while chunk i
    is copied host->device, chunk i+1 is read from the file.
    """
    dev = _device(device)
    with open(path, "rb", buffering=0) as handle:
        dim, arity, nv, ne = _read_header(handle, path)
        vb, eb = dim * 4 * nv, arity * 4 * ne
        _check_payload(handle, path, vb + eb)
        with torch.cuda.device(dev):
            buf = torch.empty(max(vb + eb, 4), dtype=torch.uint8, device=dev)
            total = vb + eb
            if total:
                size = min(chunk, total)
                stage = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
                done = [torch.cuda.Event(), torch.cuda.Event()]
                used = [False, False]
                copy = torch.cuda.Stream(dev)
                off = 0
                k = 0
                while off < total:
                    n = min(size, total - off)
                    s = k & 1
                    if used[s]:
                        done[s].synchronize()  # the staging buffer's previous copy has left
                    _readinto_exact(handle, memoryview(stage[s].numpy())[:n], path)
                    with torch.cuda.stream(copy):
                        buf[off:off + n].copy_(stage[s][:n], non_blocking=True)
                        done[s].record(copy)
                    used[s] = True
                    off += n
                    k += 1
                torch.cuda.current_stream(dev).wait_stream(copy)
                copy.synchronize()
        vtx = buf[:vb].view(torch.int32).view(nv, dim)
        idx = buf[vb:vb + eb].view(torch.int32).view(ne, arity)
    return vtx, idx


def save_bin_tensors(vertex_bits: torch.Tensor, elements: torch.Tensor, path) -> None:
    """Device (or host) int32 tensors -> RMX1 file."""
    v = vertex_bits.cpu().numpy().view("<f4")
    e = elements.cpu().numpy().view("<u4")
    with open(path, "wb") as handle:
        handle.write(HEADER.pack(MAGIC, v.shape[1], e.shape[1], v.shape[0], e.shape[0]))
        handle.write(_bytes(np.ascontiguousarray(v)))
        handle.write(_bytes(np.ascontiguousarray(e)))


def reindex_file(src, dst, device=None) -> int:
    """RMX1 file -> re-index on the device -> RMX1 file; returns the vertex count written."""
    from .pipeline import reindex_tensors
    vtx, idx = load_bin_tensors(src, device)
    if idx.shape[0] == 0:
        save_bin_tensors(vtx[:0], idx, dst)
        return 0
    res = reindex_tensors(vtx, idx)
    save_bin_tensors(res.vertices, res.elements, dst)
    return int(res.vertices.shape[0])


__all__ = ["FormatError", "read_bin", "write_bin", "load_bin_tensors", "save_bin_tensors", "reindex_file"]
