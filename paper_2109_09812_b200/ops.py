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
    """Re-indexed concatenation of meshes sharing dim and arity (ops.py:10-35).

    Each mesh is validated, uploaded, and the concatenation + index shift +
    re-index run on the device (:func:`merge_tensors`).
    """
    parts = list(meshes)
    if len(parts) == 0:
        raise MeshError("merge of an empty list of meshes")
    d0, k0 = parts[0].dim, parts[0].arity
    for pos, part in enumerate(parts):
        if (part.dim, part.arity) != (d0, k0):
            raise MeshError(f"merge: mesh #{pos} is dim {part.dim} / arity {part.arity}, "
                            f"the first mesh is dim {d0} / arity {k0}")
        require_valid(part)
    n_vtx = sum(part.n_vertices for part in parts)
    if n_vtx >= MAX_VERTICES:
        raise MeshError(f"merge: {n_vtx} vertices in total do not fit 32-bit indices")
    if sum(part.n_elements for part in parts) == 0:
        return Mesh.empty(dim=d0, arity=k0)
    dev = _device(device)
    with torch.cuda.device(dev):
        on_device = []
        for part in parts:
            v = torch.empty((part.n_vertices, d0), dtype=torch.int32, device=dev)
            e = torch.empty((part.n_elements, k0), dtype=torch.int32, device=dev)
            if part.n_vertices:
                hostio.to_device(np.ascontiguousarray(part.vertices), v)
            if part.n_elements:
                hostio.to_device(np.ascontiguousarray(part.elements), e)
            on_device.append((v, e))
        return _to_mesh(merge_tensors(on_device, dev))


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
    """Compact mesh from a (m, K, D) soup (ops.py:38-56): every element corner is a
    vertex slot of its own, element e = slots (eK .. eK+K-1), then re-index."""
    try:
        corners = np.asarray(soup, dtype=np.float32)
    except (ValueError, TypeError) as exc:
        raise MeshError(f"soup is not a rectangular (elements, arity, dim) array: {exc}") from None
    if corners.ndim != 3:
        raise MeshError(f"soup needs shape (elements, arity, dim); got {corners.shape}")
    n_el, k, d = corners.shape
    if n_el == 0:
        return Mesh.empty(dim=d, arity=k)
    slots = n_el * k
    if slots >= MAX_VERTICES:
        raise MeshError(f"soup: {slots} corners do not fit 32-bit indices")
    dev = _device(device)
    with torch.cuda.device(dev):
        vtx = torch.empty((slots, d), dtype=torch.int32, device=dev)
        hostio.to_device(np.ascontiguousarray(corners.reshape(slots, d)), vtx)
        iota = torch.arange(slots, dtype=torch.int64, device=dev).view(n_el, k)
        res = reindex_tensors(vtx, iota.to(torch.int32) if slots < (1 << 31) else _narrow_u32(iota))
    return _to_mesh(res)


def subset(mesh, keep, device=None) -> Mesh:
    """Compact mesh of the selected elements only (ops.py:59-68)."""
    require_valid(mesh)
    mask = _selector_mask(keep, len(mesh.elements))
    sub = Mesh(np.asarray(mesh.vertices), np.asarray(mesh.elements)[mask])
    return reindex(sub, device)[0]


def subset_tensors(vertex_bits: torch.Tensor, elements: torch.Tensor, keep: torch.Tensor):
    """Device-resident subset (ops.py:59-68): ``keep`` is a device bool mask over the elements
    or strictly increasing element positions; the selected elements are compacted on the device
    (``rmx_select_elements``) and re-indexed.  Returns a DeviceResult."""
    from . import _native
    E, K = elements.shape
    dev = elements.device
    with torch.cuda.device(dev):
        if keep.dtype == torch.bool:
            if keep.shape != (E,):
                raise MeshError(f"boolean selector has {tuple(keep.shape)} entries for {E} elements")
            mask = keep.to(device=dev, dtype=torch.uint8)
        else:
            pos = keep.reshape(-1).to(device=dev, dtype=torch.int64)
            if pos.numel():
                if bool((pos < 0).any()) or bool((pos >= E).any()):
                    raise MeshError(f"element positions must lie in [0, {E})")
                if pos.numel() > 1 and bool((pos[1:] <= pos[:-1]).any()):
                    raise MeshError("element positions must be strictly increasing (no repeats)")
            mask = torch.zeros(E, dtype=torch.uint8, device=dev)
            mask[pos] = 1
        lib = _native.lib()
        elements = elements.contiguous()
        out = torch.empty((E, K), dtype=elements.dtype, device=dev)
        kept = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = torch.empty(max(1, int(lib.rmx_select_workspace_bytes(E))), dtype=torch.uint8, device=dev)
        _native.check(lib.rmx_select_elements(elements.data_ptr() if E else None, E, K,
                                              mask.data_ptr() if E else None, out.data_ptr() if E else None,
                                              kept.data_ptr(), ws.data_ptr(), ws.numel(),
                                              torch.cuda.current_stream(dev).cuda_stream))
        n_kept = int(kept.item())
        return reindex_tensors(vertex_bits, out[:n_kept])


def _selector_mask(keep, n_elements: int) -> np.ndarray:
    """Element selector -> bool mask (ops.py:71-87 semantics): a bool mask of length
    n_elements, or strictly increasing element positions."""
    picks = np.asarray(keep)
    if picks.dtype == np.bool_:
        if picks.shape[0] != n_elements:
            raise MeshError(f"boolean selector has {picks.shape[0]} entries for {n_elements} elements")
        return picks
    picks = picks.ravel()
    chosen = np.zeros(n_elements, dtype=np.bool_)
    if picks.size == 0:
        return chosen
    if picks.dtype.kind not in "iu":
        raise MeshError(f"element selector of dtype {picks.dtype}: expected bools or integer positions")
    first, last = int(picks.min()), int(picks.max())
    if first < 0 or last >= n_elements:
        raise MeshError(f"element positions must lie in [0, {n_elements}); got {first}..{last}")
    pos = picks.astype(np.int64)
    if pos.size > 1 and bool(np.any(pos[1:] <= pos[:-1])):
        raise MeshError("element positions must be strictly increasing (no repeats)")
    chosen[pos] = True
    return chosen
