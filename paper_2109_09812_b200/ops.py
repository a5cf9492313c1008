"""Mesh composition on the GPU path: merge, soup_to_mesh, subset.

Same contracts as the reference (``pkg/src/remeshx/ops.py``):

* ``merge(meshes)``      ops.py:10-35 -- concatenate vertex arrays, offset each
  mesh's indices, re-index; output soup = concatenation of the input soups.
* ``soup_to_mesh(soup)`` ops.py:38-56 -- (m, K, D) value-carrying elements ->
  compact indexed mesh.
* ``subset(mesh, keep)`` ops.py:59-87 -- keep a bool mask or strictly ascending
  positions of elements, drop vertices that became unused.

Inputs are assembled directly in device memory (vertex words copied slice by
slice, element offsets added on the device) and re-indexed by the CUDA
pipeline; results come back as the package's :class:`Mesh`.
"""
from __future__ import annotations

import numpy as np
import torch

from . import hostio
from .mesh import MAX_VERTICES, Mesh, MeshError, require_valid
from .pipeline import _device, host_tensor, reindex, reindex_tensors


def _to_mesh(res) -> Mesh:
    v = hostio.to_host(res.vertices).view(np.float32)
    e = hostio.to_host(res.elements).view(np.uint32)
    return Mesh._adopt(v, e)


def merge(meshes, device=None) -> Mesh:
    """Re-indexed concatenation of meshes sharing dim and arity (ops.py:10-35)."""
    meshes = list(meshes)
    if not meshes:
        raise MeshError("merge needs at least one mesh")
    dim, arity = meshes[0].dim, meshes[0].arity
    for k, m in enumerate(meshes):
        if m.dim != dim or m.arity != arity:
            raise MeshError(f"mesh {k} has dim={m.dim} arity={m.arity}, expected dim={dim} arity={arity}")
        require_valid(m)
    total = sum(m.n_vertices for m in meshes)
    if total >= MAX_VERTICES:
        raise MeshError(f"merged vertex count {total} exceeds 32-bit index range")
    n_elem = sum(m.n_elements for m in meshes)
    if n_elem == 0:
        return Mesh.empty(dim=dim, arity=arity)
    dev = _device(device)
    with torch.cuda.device(dev):
        vtx = torch.empty((total, dim), dtype=torch.int32, device=dev)
        idx = torch.empty((n_elem, arity), dtype=torch.int64, device=dev)
        v0 = e0 = 0
        for m in meshes:
            nv, ne = m.n_vertices, m.n_elements
            if nv:
                vtx[v0:v0 + nv].copy_(host_tensor(np.ascontiguousarray(m.vertices).view(np.int32)))
            if ne:
                seg = host_tensor(np.ascontiguousarray(m.elements).view(np.int32)).to(dev)
                idx[e0:e0 + ne] = (seg.to(torch.int64) & 0xFFFFFFFF) + v0
            v0 += nv
            e0 += ne
        # offsets stay below 2**32 (checked above); narrow to the pipeline's 32-bit words
        res = reindex_tensors(vtx, idx.to(torch.int32) if total < (1 << 31) else _narrow_u32(idx))
    return _to_mesh(res)


def merge_tensors(pieces, device=None):
    """Device-resident merge (ops.py:10-35): concatenate the pieces' vertex bits,
    shift each piece's indices by the vertices before it (``rmx_offset_indices``),
    re-index.  ``pieces`` = [(vertex bits int32 (V_k, D), elements int32 (E_k, K))]
    on one device; returns the :class:`~paper_2109_09812_b200.DeviceResult`.
    """
    from . import _native
    pieces = list(pieces)
    if not pieces:
        raise MeshError("merge needs at least one mesh")
    D, K = pieces[0][0].shape[1], pieces[0][1].shape[1]
    for k, (v, e) in enumerate(pieces):
        if v.dim() != 2 or e.dim() != 2 or v.shape[1] != D or e.shape[1] != K:
            raise MeshError(f"piece {k} has shapes {tuple(v.shape)} / {tuple(e.shape)}, expected (*, {D}) / (*, {K})")
    total = sum(v.shape[0] for v, _ in pieces)
    if total >= MAX_VERTICES:
        raise MeshError(f"merged vertex count {total} exceeds 32-bit index range")
    n_elem = sum(e.shape[0] for _, e in pieces)
    dev = pieces[0][0].device if device is None else torch.device(device)
    lib = _native.lib()
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        vtx = torch.empty((total, D), dtype=torch.int32, device=dev)
        idx = torch.empty((n_elem, K), dtype=torch.int32, device=dev)
        v0 = e0 = 0
        for v, e in pieces:
            nv, ne = v.shape[0], e.shape[0]
            if nv:
                vtx[v0:v0 + nv].copy_(v, non_blocking=True)
            if ne:
                src = e.contiguous()
                _native.check(lib.rmx_offset_indices(src.data_ptr(), ne * K, v0, idx[e0:e0 + ne].data_ptr(),
                                                     stream.cuda_stream))
            v0 += nv
            e0 += ne
        return reindex_tensors(vtx, idx)


def _narrow_u32(x: torch.Tensor) -> torch.Tensor:
    """int64 values in [0, 2**32) -> int32 tensor with the same low 32 bits."""
    return (x - ((x >> 31) << 32)).to(torch.int32)


def soup_to_mesh(soup, device=None) -> Mesh:
    """Compact mesh from a (m, K, D) soup (ops.py:38-56)."""
    try:
        arr = np.asarray(soup, dtype=np.float32)
    except (ValueError, TypeError) as exc:
        raise MeshError(f"ragged soup: {exc}") from None
    if arr.ndim != 3:
        raise MeshError(f"soup must be a (m, arity, dim) array, got shape {arr.shape}")
    m, arity, dim = arr.shape
    if m == 0:
        return Mesh.empty(dim=dim, arity=arity)
    n = m * arity
    if n >= MAX_VERTICES:
        raise MeshError(f"soup has {n} vertices, exceeds 32-bit index range")
    dev = _device(device)
    with torch.cuda.device(dev):
        vtx = host_tensor(np.ascontiguousarray(arr.reshape(n, dim)).view(np.int32)).to(dev)
        idx = torch.arange(n, dtype=torch.int64, device=dev).view(m, arity)
        res = reindex_tensors(vtx, idx.to(torch.int32) if n < (1 << 31) else _narrow_u32(idx))
    return _to_mesh(res)


def subset(mesh, keep, device=None) -> Mesh:
    """Compact mesh of the selected elements only (ops.py:59-68)."""
    require_valid(mesh)
    mask = _selector_mask(keep, len(mesh.elements))
    sub = Mesh(np.asarray(mesh.vertices), np.asarray(mesh.elements)[mask])
    return reindex(sub, device)[0]


def _selector_mask(keep, n_elements: int) -> np.ndarray:
    """Bool mask or strictly ascending positions -> mask (ops.py:71-87)."""
    sel = np.asarray(keep)
    if sel.dtype == bool:
        if len(sel) != n_elements:
            raise MeshError(f"mask length {len(sel)} != element count {n_elements}")
        return sel
    sel = sel.reshape(-1)
    if sel.size:
        if not np.issubdtype(sel.dtype, np.integer):
            raise MeshError(f"selector must be a bool mask or integer positions, got {sel.dtype}")
        if int(sel.min()) < 0 or int(sel.max()) >= n_elements:
            raise MeshError(f"selector position out of range [0, {n_elements})")
        if sel.size > 1 and not bool(np.all(sel[1:] > sel[:-1])):
            raise MeshError("selector positions must be strictly ascending and unique")
    mask = np.zeros(n_elements, dtype=bool)
    mask[sel.astype(np.int64)] = True
    return mask
