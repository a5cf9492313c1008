"""ctypes binding of the C-ABI in ``include/remesh_b200.h``.

The shared library ``librmx_b200.so`` is built in-tree by
``paper_2109_09812_b200.build.build()`` (nvcc, ``-gencode
arch=compute_100a,code=sm_100a``).  There is deliberately no fallback: if the
library is missing every entry point raises :class:`NativeLibraryMissing`.
Loading the library needs no GPU (cudart is linked statically), so symbol
checks run on CPU-only machines.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "librmx_b200.so"
# RMX_LIB overrides the library file (tuning builds, e.g. the -DRMX_PHASES variant)
LIB_PATH = os.environ.get("RMX_LIB") or os.path.join(_HERE, LIB_NAME)

RMX_OK, RMX_EINVAL, RMX_ERANGE, RMX_ECUDA, RMX_ENOSPC = 0, 1, 2, 3, 4
RMX_STATUS_INDEX_OUT_OF_RANGE = 1
RMX_STATUS_LEAN_UNSUPPORTED = 2
RMX_MAX_DIM = 32

# every symbol include/remesh_b200.h declares
EXPORTS = (
    "rmx_version", "rmx_strerror", "rmx_workspace_bytes", "rmx_reindex", "rmx_lean_workspace_bytes",
    "rmx_lean_result_offset", "rmx_reindex_lean",
    "rmx_reindex_profiled", "rmx_stage_count", "rmx_stage_name", "rmx_kernel_launches", "rmx_kernel_launches_total", "rmx_debug_oob_count",
    "rmx_last_executed_passes", "rmx_plan_info", "rmx_plan_key_info", "rmx_plan_guess_info", "rmx_hash_info", "rmx_soup_info", "rmx_window_info", "rmx_debug_phase_cycles", "rmx_lattice_sizes",
    "rmx_gen_lattice_soup", "rmx_gen_lattice_soup_range", "rmx_gen_grid_quads", "rmx_gather_u32", "rmx_lower_bound_rows",
    "rmx_graph_create", "rmx_graph_launch", "rmx_graph_destroy", "rmx_offset_indices",
    "rmx_welded_tile_sizes", "rmx_gen_welded_tile", "rmx_scatter_rows", "rmx_merge_workspace_bytes",
    "rmx_merge_unique_runs", "rmx_select_workspace_bytes", "rmx_select_elements",
)


class NativeLibraryMissing(RuntimeError):
    """The CUDA library is not built; run ``python -c 'import __graft_entry__ as g; g.build()'``."""


class Scratch(ctypes.Structure):
    """``rmx_scratch`` (device pointers, NULL = not requested)."""

    _fields_ = [("is_used", ctypes.c_void_p), ("org_id", ctypes.c_void_p),
                ("nodup", ctypes.c_void_p), ("new_idx", ctypes.c_void_p),
                ("perm", ctypes.c_void_p)]


_lock = threading.Lock()
_lib = None

_vp, _u64, _u32, _sz, _int = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                              ctypes.c_size_t, ctypes.c_int)

_SIGNATURES = {
    "rmx_version": (ctypes.c_char_p, []),
    "rmx_strerror": (ctypes.c_char_p, [_int]),
    "rmx_workspace_bytes": (_sz, [_u64, _u32, _u64, _u32]),
    "rmx_lean_workspace_bytes": (_sz, [_u64, _u32, _u64, _u32]),
    "rmx_lean_result_offset": (_sz, [_u64, _u32]),
    "rmx_reindex_lean": (_int, [_vp, _u64, _u32, _vp, _u64, _u32, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "rmx_reindex": (_int, [_vp, _u64, _u32, _vp, _u64, _u32, _vp, _vp, _vp, _vp, _vp, _sz,
                           ctypes.POINTER(Scratch), _vp]),
    "rmx_reindex_profiled": (_int, [_vp, _u64, _u32, _vp, _u64, _u32, _vp, _vp, _vp, _vp, _vp, _sz,
                                    ctypes.POINTER(Scratch), _vp, ctypes.POINTER(_vp), _int]),
    "rmx_stage_count": (_int, [_u32]),
    "rmx_kernel_launches": (_int, [_u32]),
    "rmx_kernel_launches_total": (ctypes.c_ulonglong, []),
    "rmx_debug_oob_count": (_int, [ctypes.POINTER(ctypes.c_ulonglong)]),
    "rmx_stage_name": (ctypes.c_char_p, [_u32, _int]),
    "rmx_last_executed_passes": (_int, [_vp, _u64, _u32, _vp]),
    "rmx_plan_info": (_int, [_vp, _u64, _u32, _vp, ctypes.POINTER(_u32)]),
    "rmx_plan_key_info": (_int, [_vp, _u64, _u32, _vp, ctypes.POINTER(_u32)]),
    "rmx_plan_guess_info": (_int, [_vp, _u64, _u32, _vp, ctypes.POINTER(_u32)]),
    "rmx_hash_info": (_int, [_vp, _u64, _u32, _vp, ctypes.POINTER(_u32)]),
    "rmx_soup_info": (_int, [_vp, _u64, _u32, _vp, ctypes.POINTER(_u32)]),
    "rmx_window_info": (_int, [_vp, _u64, _u32, _vp, ctypes.POINTER(_u32)]),
    "rmx_debug_phase_cycles": (_int, [ctypes.POINTER(ctypes.c_ulonglong), _int, _int]),
    "rmx_lattice_sizes": (_int, [_int, _u32, _u32, _u32, _u64,
                                 ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "rmx_gen_lattice_soup": (_int, [_int, _u32, _u32, _u32, _u64, _u64, _vp, _vp, _vp]),
    "rmx_gen_lattice_soup_range": (_int, [_int, _u32, _u32, _u32, _u64, _u64, _u64, _vp, _vp, _vp]),
    "rmx_gen_grid_quads": (_int, [_u32, _vp, _vp, _vp]),
    "rmx_gather_u32": (_int, [_vp, _u64, _vp, _u64, _vp, _vp, _vp]),
    "rmx_lower_bound_rows": (_int, [_vp, _u64, _u32, _vp, _u64, _vp, _vp]),
    "rmx_graph_create": (_int, [_vp, _u64, _u32, _vp, _u64, _u32, _vp, _vp, _vp, _vp, _vp, _sz,
                                ctypes.POINTER(Scratch), ctypes.POINTER(_vp)]),
    "rmx_graph_launch": (_int, [_vp, _vp]),
    "rmx_graph_destroy": (None, [_vp]),
    "rmx_offset_indices": (_int, [_vp, _u64, _u32, _vp, _vp]),
    "rmx_welded_tile_sizes": (_int, [_u32, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "rmx_gen_welded_tile": (_int, [_u32, _u32, _u64, _int, _vp, _vp, _vp]),
    "rmx_scatter_rows": (_int, [_vp, _u64, _u32, _vp, _u32, _vp, _vp, _vp]),
    "rmx_merge_workspace_bytes": (_sz, [_u64, _u32]),
    "rmx_select_workspace_bytes": (_sz, [_u64]),
    "rmx_select_elements": (_int, [_vp, _u64, _u32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "rmx_merge_unique_runs": (_int, [_vp, _u64, _u32, ctypes.POINTER(_u64), _u32, _vp, _vp, _vp, _vp, _sz, _vp]),
}


def lib():
    """The loaded library; raises :class:`NativeLibraryMissing` if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not found: the CUDA re-indexing library is not built "
                    "(there is no CPU fallback). Build it with paper_2109_09812_b200.build.build().")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(rc: int) -> None:
    """Raise for a non-zero C-ABI return code (mapping in pipeline._raise_for)."""
    if rc != RMX_OK:
        msg = lib().rmx_strerror(rc).decode()
        raise NativeError(rc, msg)


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        self.code = code
        super().__init__(f"rmx error {code}: {message}")
